/* gplan.h — C ABI of the B200 plan-evaluation engine (libgplan.so).
 *
 * Drop-in boundary for the hot path of the rlsched reference scheduler
 * (arXiv 2511.00796, /root/reference/proj). The reference has no plugin
 * registry: its seam is the C++ free-function API that
 * `partition_with_widening` / `evaluate_partition` call (src/scheduler.cpp:21-40,
 * 42-75). Each entry point below replaces exactly one of
 * those functions; the C++ shim in paper_2511_00796_b200/shim/ re-exposes them
 * under the reference signatures so the reference scheduler.cpp links
 * unchanged.
 *
 * Conventions
 *   - Plain pointers and sizes only; caller owns every input buffer (borrowed
 *     for the duration of the call) and every output buffer.
 *   - No exceptions cross the ABI. Every function returns a gp_status; the
 *     C++ shim rethrows the matching rlsched exception (inc/common.hpp:11-39).
 *   - Calls are synchronous and blocking; one host thread per context.
 *   - All arithmetic is IEEE fp64 without contraction and reproduces the
 *     reference bit-for-bit.
 *   - A context owns its CUDA device buffers and stream; there is no CPU
 *     fallback: if the CUDA device or the kernels are unavailable,
 *     gp_ctx_create fails with GP_CUDA_ERROR.
 */
#ifndef GPLAN_H_
#define GPLAN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GP_ABI_VERSION 1

/* Limits of the fixed-size result records. */
#define GP_MAX_TYPES 8           /* gpu types in one cluster                          */
#define GP_MAX_STAGES 32         /* pipeline stages of a train plan (4 per type run)  */
#define GP_MAX_ROLLOUT_STAGES 8  /* pipeline stages of one rollout replica config     */

typedef enum {
  GP_OK = 0,
  GP_INFEASIBLE = 1,       /* rlsched::InfeasibleError       */
  GP_BAND_INFEASIBLE = 2,  /* rlsched::BandInfeasibleError   */
  GP_INVALID = 3,          /* rlsched::ValidationError       */
  GP_CUDA_ERROR = 4,       /* device/runtime failure (no fallback) */
  GP_CAPACITY = 5          /* caller-provided output buffer too small */
} gp_status;

/* ---- inputs (mirror inc/cluster.hpp:16-59, inc/workload.hpp:43-66,
 *      inc/calibration.hpp:15-33) ---------------------------------------- */

/* ClusterGraph (inc/cluster.hpp:40-63) flattened to SoA. SI units. */
typedef struct {
  int32_t n_devices;
  int32_t n_types;
  int32_t n_machines;
  const int32_t* device_type;     /* [n_devices] GpuDevice::gpu_type            */
  const int32_t* device_machine;  /* [n_devices] GpuDevice::machine_id          */
  const double* device_flops;     /* [n_devices] GpuDevice::flops               */
  const double* device_hbm_bw;    /* [n_devices] GpuDevice::hbm_bandwidth       */
  const double* device_hbm_cap;   /* [n_devices] GpuDevice::hbm_capacity        */
  const double* type_flops;       /* [n_types]   GpuTypeInfo::flops             */
  const double* type_hbm_bw;      /* [n_types]   GpuTypeInfo::hbm_bandwidth     */
  const double* type_hbm_cap;     /* [n_types]   GpuTypeInfo::hbm_capacity      */
  const double* links;            /* [n_devices^2] row-major, bytes/s           */
} gp_cluster;

/* WorkloadSpec scalars (inc/workload.hpp:43-66). */
typedef struct {
  double model_params_b;
  int32_t num_layers;
  int32_t hidden_dim;
  int32_t batch_rollouts;
  int32_t prompt_len;
  double mean_len;                /* LengthDistribution::mean()                 */
  double bytes_per_param_train;
  double bytes_per_param_infer;
  double reward_cost_const;
  int32_t micro_batches;
  int32_t staleness;
} gp_workload;

/* Calibration (inc/calibration.hpp:15-33), per-type efficiencies by type index. */
typedef struct {
  const double* compute_eff;      /* [n_types] */
  const double* io_eff;           /* [n_types] */
  double sync_latency_s;
  double stage_latency_penalty;
  int32_t max_concurrency;
  double activation_coeff;
  double tp_allreduce_coeff;
  double grad_bytes_per_param;
} gp_calib;

/* ---- options (inc/train_search.hpp:12-17, inc/rollout_milp.hpp:14-16,
 *      inc/partition.hpp:10-30) ---------------------------------------------- */
typedef struct {
  int32_t max_stages_per_type;       /* default 4  */
  int32_t device_granularity_limit;  /* default 16 */
} gp_train_opts;

typedef struct {
  int32_t max_stages;                /* default 4 (<= GP_MAX_ROLLOUT_STAGES) */
} gp_rollout_opts;

typedef struct {
  double q, r, gamma_l, gamma_h;     /* GammaState */
} gp_gamma;

typedef struct {
  int32_t exact_threshold;           /* default 12     */
  int32_t restarts;                  /* default 16     */
  uint64_t seed;                     /* default 0x5eed */
  double band_epsilon;               /* default 1e-9   */
  int32_t force_local_search;
  int32_t machine_granularity;
} gp_part_opts;

/* ---- results --------------------------------------------------------------- */

typedef struct {
  int32_t first;   /* offset into the caller's stage_devices buffer */
  int32_t count;   /* tp * dp                                       */
  int32_t tp, dp, layers;
} gp_stage;

/* std::optional<TrainSearchResult> (inc/train_search.hpp:19-33). */
typedef struct {
  int32_t found;          /* 0 == std::nullopt: no memory-feasible layout   */
  int32_t n_stages;
  double cost;            /* C_T = window * per_step (TrainSearchResult::cost) */
  int64_t rank;           /* rank of the winner in the reference enumeration order */
  int64_t layouts;        /* candidate layouts evaluated (the range size)   */
  int64_t feasible;       /* memory-feasible layouts among them             */
  gp_stage stage[GP_MAX_STAGES];
} gp_train_result;

/* ReplicaConfig (inc/plans.hpp:47-66); machine_footprint == tp_per_stage. */
typedef struct {
  int32_t type_counts[GP_MAX_TYPES];
  int32_t n_stages;
  int32_t tp[GP_MAX_ROLLOUT_STAGES];
  double throughput;
} gp_config;

typedef struct {
  int32_t config;         /* index into the config list passed to gp_solve_milp */
  int32_t replicas;       /* y */
  double workload;        /* x */
} gp_rollout_entry;

/* RolloutPlan (inc/plans.hpp:75-85). entries is caller-provided. */
typedef struct {
  int32_t n_entries;
  double makespan;
  double total_rollouts;
  double aggregate;       /* best[full state] */
  int64_t states;         /* lattice size */
} gp_rollout_result;

/* PartitionResult (inc/partition.hpp:32-36); train ids are written to a
 * caller buffer at train_offset. */
typedef struct {
  int32_t train_offset;
  int32_t train_count;
  double objective;
  double compute_fraction;
} gp_partition;

typedef struct gp_ctx gp_ctx;

/* ---- lifecycle ------------------------------------------------------------- */

/* Validates and uploads the cluster/workload/calibration to `device`
 * (CUDA ordinal). Fails with GP_CUDA_ERROR when no usable sm_100 device or
 * kernel image exists. */
int gp_ctx_create(const gp_cluster* cluster, const gp_workload* work, const gp_calib* calib,
                  int device, gp_ctx** out);
/* Multi-GPU context: the same inputs on every listed CUDA ordinal. Searches whose
 * layout range is large are split into contiguous rank shards, one per device, run
 * concurrently and reduced lexicographically inside the call; every other entry point
 * runs on devices[0]. */
int gp_ctx_create_multi(const gp_cluster* cluster, const gp_workload* work, const gp_calib* calib,
                        const int* devices, int n_devices, gp_ctx** out);
void gp_ctx_destroy(gp_ctx* ctx);
/* Message of the last failing call on this thread. */
const char* gp_last_error(void);
int gp_abi_version(void);
/* Kernel launches issued by this context so far (diagnostics / bench claim). */
long long gp_ctx_launches(gp_ctx* ctx);

/* ---- training side: replaces constrained_search (src/train_search.cpp:218-275) */

/* Number of layouts constrained_search would enumerate for `ids`
 * (enumerate_block_lists, src/train_search.cpp:126-142), without materialising. */
int gp_train_space(gp_ctx* ctx, const int32_t* ids, int32_t n, const gp_train_opts* opts,
                   int64_t* layouts);

/* constrained_search(train_set, cluster, work, calib, window, options)
 * (inc/train_search.hpp:29-33). stage_devices must hold n ints; stage s owns
 * stage_devices[stage[s].first .. +count). Empty train set -> GP_INVALID.
 * The scan is window-independent: each train set's near-minimum summary is
 * memoised on the context, and a later call for the same set with another
 * window is answered from it bit-exactly (gp_ctx_set_memo(ctx, 0) disables). */
int gp_constrained_search(gp_ctx* ctx, const int32_t* ids, int32_t n, int32_t window,
                          const gp_train_opts* opts, gp_train_result* out,
                          int32_t* stage_devices);

/* Same search restricted to layout ranks [lo, hi): the shard one GPU scans in
 * the multi-GPU split. The global winner is the lexicographic
 * min of (cost, rank) over shards. */
int gp_constrained_search_range(gp_ctx* ctx, const int32_t* ids, int32_t n, int32_t window,
                                const gp_train_opts* opts, int64_t lo, int64_t hi,
                                gp_train_result* out, int32_t* stage_devices);

/* Many constrained_search calls in one (the scheduler's evaluation batches, SURVEY 8f
 * rank 1): set i is ids[off[i] .. off[i+1]) and its result goes to out[i] (its stage
 * devices to stage_devices[off[i] ..]). All inputs travel in one H2D copy, every set's
 * tables and scan are in flight together (small sets fused, one CTA each), results come
 * back in one D2H copy; memoised like gp_constrained_search; split over the devices of a
 * multi-device context by layout count. */
int gp_constrained_search_batch(gp_ctx* ctx, int32_t n_sets, const int32_t* ids, const int32_t* off,
                                int32_t window, const gp_train_opts* opts, gp_train_result* out,
                                int32_t* stage_devices);

/* Split form of gp_constrained_search_range for callers that overlap work or
 * time the device part alone (bench.py): prepare uploads the train set's
 * enumeration metadata (one H2D copy), launch enqueues the stage-table build
 * and the layout scan on the context's stream without blocking, collect
 * copies the result back and synchronises. */
int gp_train_prepare(gp_ctx* ctx, const int32_t* ids, int32_t n, const gp_train_opts* opts);
int gp_train_launch(gp_ctx* ctx, int32_t window, int64_t lo, int64_t hi);
int gp_train_collect(gp_ctx* ctx, gp_train_result* out, int32_t* stage_devices);
/* The context's CUDA stream (cudaStream_t), for event timing by the caller. */
void* gp_ctx_stream(gp_ctx* ctx);
/* Measurement hooks (bench.py): device time of the last launch's stage-table
 * build (K2) and layout scan (K1 + finalize); bytes moved host<->device by API
 * calls so far; sum over the prepared space of the stage count; FP64 pipe
 * throughput probe (DADD/s) used as the roofline denominator. */
int gp_ctx_set_timing(gp_ctx* ctx, int on);
/* Enable (default) / disable + drop the constrained_search memo. */
int gp_ctx_set_memo(gp_ctx* ctx, int on);
int gp_train_timing(gp_ctx* ctx, float* k2_ms, float* k1_ms);
void gp_ctx_io_bytes(gp_ctx* ctx, long long* h2d, long long* d2h, double* sum_stages);
int gp_fp64_peak(gp_ctx* ctx, double* dadd_per_s);
/* Test hook (parity of individual candidates, not a reference interface): per_step
 * (train_cost_breakdown(...).per_step, src/cost_model.cpp:93-126) of every layout of
 * ranks [lo, hi) of the train set, computed by the scan kernel itself (its DUMP
 * instantiation), +inf for layouts without a memory-feasible option. path 0: the
 * whole-space scan constrained_search runs (K1-fast with its inner run when eligible), the
 * values of [lo, hi) kept; 1: the generic K1 over [lo, hi); 2: K1-fast over [lo, hi) with
 * every candidate deferred to its generic fallback; 3: K1-fast over [lo, hi) as a range
 * search scans it. hi - lo <= 2^26. *fast_used (optional): 1 + K1-fast's inner type run,
 * 0 when the generic K1 scored the range. */
int gp_debug_layout_costs(gp_ctx* ctx, const int32_t* ids, int32_t n, const gp_train_opts* opts,
                          int64_t lo, int64_t hi, int32_t path, double* per_step, int32_t* fast_used);
/* Rank boundaries bounds[0..n_shards] splitting a train set's layout space into n_shards
 * contiguous ranges of equal size for multi-GPU sharding (gp_constrained_search_range per
 * shard, winners merged by (cost, rank), feasible counts summed). */
int gp_train_shard_bounds(gp_ctx* ctx, const int32_t* ids, int32_t n, const gp_train_opts* opts,
                          int32_t n_shards, int64_t* bounds);

/* ---- rollout side: replaces enumerate_configs / rollout_capacities / solve_milp
 *      (src/rollout_milp.cpp:30-171) ------------------------------------- */

/* enumerate_configs (inc/rollout_milp.hpp:22-25, src/rollout_milp.cpp:39-89); out holds cap
 * records; GP_CAPACITY with *n_out = the count needed when cap is too small. */
int gp_enumerate_configs(gp_ctx* ctx, const int32_t* ids, int32_t n, const gp_rollout_opts* opts,
                         gp_config* out, int32_t cap, int32_t* n_out);
/* rollout_capacities (inc/rollout_milp.hpp:28-29, src/rollout_milp.cpp:30-37). */
int gp_rollout_capacities(gp_ctx* ctx, const int32_t* ids, int32_t n, int32_t* caps);
/* Many solve_milp instances in one call (the scheduler's evaluation batches): query i has
 * configs[cfg_off[i] .. cfg_off[i+1]), caps[i*dims ..], total_rollouts[i]; results in
 * out[i], entries at entries[cfg_off[i] ..], status per query in status[i] (GP_OK,
 * GP_INFEASIBLE, GP_INVALID). The lattice DPs of all queries run batched. */
int gp_solve_milp_batch(gp_ctx* ctx, int32_t q, const gp_config* configs, const int32_t* cfg_off,
                        const int32_t* caps, int32_t dims, const double* total_rollouts, double mean_len,
                        gp_rollout_result* out, gp_rollout_entry* entries, int32_t* status);
/* solve_milp (inc/rollout_milp.hpp:35-37, src/rollout_milp.cpp:91-171): the exact makespan
 * DP. entries must hold n_configs records. B <= 0 -> empty plan. */
int gp_solve_milp(gp_ctx* ctx, const gp_config* configs, int32_t n_configs, const int32_t* caps,
                  int32_t dims, double total_rollouts, double mean_len, gp_rollout_result* out,
                  gp_rollout_entry* entries);

/* ---- weight sync: replaces weight_sync_cost (inc/cost_model.hpp:63-65,
 *      src/cost_model.cpp:174-196) ---------------------------------------------- */
int gp_weight_sync_cost(gp_ctx* ctx, const int32_t* train, int32_t n_train, const int32_t* rollout,
                        int32_t n_rollout, const int32_t* entry_types,
                        const int32_t* entry_replicas, int32_t n_entries, int32_t window,
                        double* out);

/* ---- repartition: replaces graph_partition_candidates (inc/partition.hpp:53-55,
 *      src/partition.cpp:369-406) -------------------------------------------- */
/* out holds up to k records; train_ids holds up to k * n_devices ints. */
int gp_partition_candidates(gp_ctx* ctx, const gp_gamma* gamma, const gp_part_opts* opts,
                            int32_t k, gp_partition* out, int32_t* train_ids, int32_t* n_out);
/* partition_objective (inc/partition.hpp:40-42, src/partition.cpp:354-358). */
int gp_partition_objective(gp_ctx* ctx, const int32_t* train, int32_t n_train, double* objective,
                           double* fraction);
/* compute_fraction (src/partition.cpp:361-367). */
int gp_compute_fraction(gp_ctx* ctx, const int32_t* train, int32_t n_train, double* fraction);

/* ---- Algorithm-1 driver on the engine: schedule() (src/scheduler.cpp:259-292) ----- */

/* SchedulerOptions (inc/scheduler.hpp:15-34) + the solver options it carries. */
typedef struct {
  int32_t eta_override;        /* < 0: the workload's staleness */
  int32_t stable_iters;        /* 20 */
  int32_t iteration_cap;       /* 200 */
  double stability_tol;        /* 0.005 */
  double balance_tol;          /* 0.02 */
  double interval_min;         /* 1e-3 */
  double band_widen_step;      /* 0.05 */
  int32_t delta_cap;           /* 64 */
  int32_t expand_window;       /* 1 */
  int32_t candidate_width;     /* 8 */
  int32_t grid_probes;         /* 15 */
  gp_train_opts train;
  gp_rollout_opts rollout;
  int32_t exact_threshold;     /* PartitionOptions: 12 */
  int32_t restarts;            /* 16 */
  uint64_t seed;               /* 0x5eed (the CLI passes 4276115) */
  double band_epsilon;         /* 1e-9 */
  int32_t force_local_search;
  int32_t machine_granularity;
} gp_sched_opts;

typedef struct {
  int32_t window, staleness, iterations_run, converged;
  int32_t n_trace;             /* IterationTrace rows (gamma_mid, c_train, c_infer, objective) */
  int32_t n_train, n_rollout;  /* partition sizes (ids in the caller's buffers) */
  gp_train_result train;       /* stage devices in the caller's stage_devices buffer */
  gp_rollout_result rollout;   /* entries[i].config indexes entry_configs */
  double c_train, c_rollout, c_reward, c_update, c_infer_total;
  int64_t evaluated_partitions, evaluated_layouts;
} gp_schedule_result;

void gp_default_sched_opts(gp_sched_opts* o);
/* train_ids, rollout_ids, stage_devices: n_devices ints each; entry_configs/entries:
 * entry_cap records; trace: 4 * iteration_cap doubles. */
int gp_schedule(gp_ctx* ctx, const gp_sched_opts* opts, gp_schedule_result* out, int32_t* train_ids,
                int32_t* rollout_ids, int32_t* stage_devices, gp_config* entry_configs,
                gp_rollout_entry* entries, int32_t entry_cap, double* trace);

/* ---- exhaustive evaluation -------------------------------- */

/* Product-space training search: every candidate of enumerate_train_candidates
 * (src/train_search.cpp:179-216; block lists x per-stage (tp, dp) options in odometer
 * order), filtered by train_plan_fits (src/cost_model.cpp:232-241), ranked by
 * train_step_cost, first minimum — the loop of tests/oracles.cpp:166-174.
 * out->layouts = candidates, out->rank = the winner's candidate index; feasible is not
 * counted (-1). Default TrainSearchOptions. */
int gp_train_candidates_search(gp_ctx* ctx, const int32_t* ids, int32_t n, int32_t window,
                               gp_train_result* out, int32_t* stage_devices);

typedef struct {
  int32_t feasible;
  int32_t n_train;            /* train_ids[0 .. n_train) ascending */
  double objective;           /* max(C_T, C_I) of the optimum */
  int64_t partitions;         /* bipartitions evaluated: 2^N - 2 */
  int64_t train_candidates;   /* product-space training candidates over all partitions */
  int64_t replica_vectors;    /* integer replica-count vectors enumerated */
} gp_exhaustive_result;

/* exhaustive_schedule_optimum (tests/oracles.cpp:144-209): over every bipartition of the
 * cluster, the product-space training optimum, enumerate_configs + brute_milp_unbounded
 * (tests/oracles.cpp:110-115, every integer replica vector), weight_sync_cost; objective
 * max(C_T, C_I), first strict minimum in mask order, preferring C_I >= C_T. The
 * reference refuses N > 10 (tests/oracles.cpp:148-151); the engine takes N <= 20.
 * train_ids: N ints. */
int gp_exhaustive_optimum(gp_ctx* ctx, int32_t window, gp_exhaustive_result* out, int32_t* train_ids);

/* ---- simulation of a scheduled plan ------------------------ */

typedef struct {
  int32_t window, staleness;          /* ScheduledPlan::window / ::staleness */
  double c_train, c_update, c_reward; /* ScheduledPlan::costs (per window) */
  int32_t n_entries;                  /* rollout_plan.entries */
  const gp_config* configs;           /* entry configs (type_counts, n_stages, tp, throughput) */
  const int32_t* replicas;            /* entry replica counts */
  int32_t n_train, n_rollout;
  const int32_t* train_ids;           /* partition.train_set (plan order) */
  const int32_t* rollout_ids;         /* partition.rollout_set (plan order) */
  const double* device_price;         /* $/hour per device id (cost reporting), n_devices */
  int32_t n_buckets;                  /* workload length histogram (length, probability) */
  const int32_t* bucket_len;
  const double* bucket_prob;
} gp_sim_plan;

typedef struct {
  int32_t steps_completed, pad;
  double avg_step_time, avg_step_time_steady, throughput_tokens_per_s;
  int64_t max_staleness_observed;
  double rollout_stall_time, trainer_wait_time, rollout_busy_time, train_busy_time;
  double sync_time_total, reward_time_total;
  int64_t rollouts_produced, rollouts_consumed, rollouts_pending, rollouts_in_flight, tokens_consumed;
  double total_time;
  double dollar_cost_per_token;       /* NaN when the throughput is 0 (std::nullopt) */
} gp_sim_report;

/* simulate (src/simulator.cpp:381-403, events not recorded) for n_seeds seeds at once,
 * one GPU thread per simulation (replica-parallel). used_devices (may be null): the
 * concrete rollout device ids bound to replicas (same for every seed), n_rollout ints;
 * n_used receives their count. GP_INVALID on the reference's ValidationErrors (no
 * replicas, too few devices, deadlock), GP_CAPACITY when a queue exceeds its bound. */
int gp_simulate(gp_ctx* ctx, const gp_sim_plan* plan, int32_t steps, int32_t sync_every, const uint64_t* seeds,
                int32_t n_seeds, gp_sim_report* out, int32_t* used_devices, int32_t* n_used);

#ifdef __cplusplus
}
#endif
#endif /* GPLAN_H_ */
