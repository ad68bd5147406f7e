/* oracle.h — TEST INFRASTRUCTURE ONLY (parity checker, never the product).
 *
 * Plain-C restatement of the rlsched reference hot path
 * (/root/reference/proj/src/{train_search,rollout_milp,cost_model,partition,scheduler}.cpp)
 * over the same SoA inputs the B200 engine takes (include/gplan.h).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load liboracle.so. Pinned against the unmodified reference
 * (oracle/_ref/libref.so) and the committed golden vectors in tests/golden/.
 */
#ifndef GP_ORACLE_H_
#define GP_ORACLE_H_

#include <stdint.h>

#include "../include/gplan.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* or_last_error(void);

int or_train_space(const gp_cluster* c, const gp_workload* w, const int32_t* ids, int32_t n,
                   const gp_train_opts* opts, int64_t* layouts);
int or_constrained_search(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                          const int32_t* ids, int32_t n, int32_t window, const gp_train_opts* opts,
                          int64_t lo, int64_t hi, gp_train_result* out, int32_t* stage_devices);

/* per_step of every layout of ranks [lo, hi) (+inf: no memory-feasible option) */
int or_layout_costs(const gp_cluster* c, const gp_workload* w, const gp_calib* k, const int32_t* ids,
                    int32_t n, const gp_train_opts* opts, int64_t lo, int64_t hi, double* per_step);
/* constrained_search over ranks [lo, hi) with memoised pure sub-results (min-links, stage
 * picks, block FLOPS), several windows in one scan, pthreads over rank chunks. out_rank[i]
 * = -1: nothing feasible. dump (optional): per_step of every rank, as or_layout_costs. */
int or_constrained_search_tab(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                              const int32_t* ids, int32_t n, const gp_train_opts* opts,
                              const int32_t* windows, int32_t n_windows, int64_t lo, int64_t hi,
                              int32_t threads, double* out_cost, int64_t* out_rank,
                              int64_t* feasible, int64_t* layouts, double* dump);

/* per_step of several rank ranges [lo[i], hi[i]) concatenated into out (tables built once) */
int or_layout_costs_tab(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                        const int32_t* ids, int32_t n, const gp_train_opts* opts, int32_t n_ranges,
                        const int64_t* lo, const int64_t* hi, double* out);

int or_enumerate_configs(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                         const int32_t* ids, int32_t n, const gp_rollout_opts* opts,
                         gp_config* out, int32_t cap, int32_t* n_out);
int or_rollout_capacities(const gp_cluster* c, const int32_t* ids, int32_t n, int32_t* caps);
int or_solve_milp(const gp_config* configs, int32_t n_configs, const int32_t* caps, int32_t dims,
                  double total_rollouts, double mean_len, gp_rollout_result* out,
                  gp_rollout_entry* entries);
int or_weight_sync_cost(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                        const int32_t* train, int32_t n_train, const int32_t* rollout,
                        int32_t n_rollout, const int32_t* entry_types,
                        const int32_t* entry_replicas, int32_t n_entries, int32_t window,
                        double* out);

int or_partition_candidates(const gp_cluster* c, const gp_gamma* g, const gp_part_opts* opts,
                            int32_t k, gp_partition* out, int32_t* train_ids, int32_t* n_out);
/* move/swap candidates examined by or_partition_candidates' local search since the last
 * reset (the U3 work unit of SURVEY 8d) */
int64_t or_partition_evals(int reset);
int or_partition_objective(const gp_cluster* c, const int32_t* train, int32_t n_train,
                           double* objective, double* fraction);

/* Algorithm 1 driver: schedule() (src/scheduler.cpp:259-292). */
typedef struct {
  int32_t eta_override;      /* < 0: use workload staleness */
  uint64_t seed;
  int32_t restarts;
  int32_t expand_window;
  double band_widen_step;    /* 0.05 */
  int32_t tab_threads;       /* > 0: large train sets via or_constrained_search_tab (threads) */
} or_sched_opts;

/* Writes a malloc'd JSON document with the plan_to_json fields (values only,
 * fingerprints omitted) + trace; free with or_free. */
int or_schedule(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                const or_sched_opts* opts, char** plan_json);
void or_free(void* p);

/* product-space training search (tests/oracles.cpp:166-174 over src/train_search.cpp:179-216):
 * out->layouts = candidates, out->feasible = candidates passing train_plan_fits,
 * out->rank = winner's candidate index */
int or_train_candidates_search(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                               const int32_t* ids, int32_t n, int32_t window, gp_train_result* out,
                               int32_t* stage_devices);
/* brute_milp_unbounded (tests/oracles.cpp:16-115); counts: n_configs ints */
int or_brute_milp(const gp_config* configs, int32_t n_configs, const int32_t* caps, int32_t dims,
                  double total_rollouts, double mean_len, int32_t* feasible, double* theta,
                  int32_t* counts, int64_t* vectors);
/* exhaustive_schedule_optimum (tests/oracles.cpp:144-209), no device-count limit */
int or_exhaustive_optimum(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                          int32_t window, gp_exhaustive_result* out, int32_t* train_ids);

#ifdef __cplusplus
}
#endif
#endif
