/* oracle.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the rlsched hot path.
 *
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). This file is the parity checker for the CUDA engine;
 * it is never linked into libgplan.so and the product never calls it.
 * Floating point: every expression keeps the reference's association order
 * and is compiled with -ffp-contract=off (no FMA), like the reference's
 * SSE2 scalar object code.
 */
#include "oracle.h"

#include <limits.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define K_INF 1e30            /* inc/common.hpp:41 */
#define K_ACT_BYTES 2.0       /* src/cost_model.cpp:10 */

static _Thread_local char g_err[512];

int or__fail(int code, const char* fmt, ...);
#define fail or__fail
int or__fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* or_last_error(void) { return g_err; }
void or_free(void* p) { free(p); }

/* ---------------------------------------------------------------- workload */
/* inc/workload.hpp:51-58 */
static double w_params(const gp_workload* w) { return w->model_params_b * 1e9; }
static double w_mean_total_len(const gp_workload* w) { return w->prompt_len + w->mean_len; }
static double w_tokens(const gp_workload* w) {
  return w->batch_rollouts * w_mean_total_len(w);
}
static double w_model_bytes_infer(const gp_workload* w) {
  return w_params(w) * w->bytes_per_param_infer;
}
static double w_kv_bytes_per_token(const gp_workload* w) {
  return 4.0 * w->hidden_dim * w->num_layers;
}

static double link(const gp_cluster* c, int a, int b) {
  return c->links[(size_t)a * (size_t)c->n_devices + (size_t)b];
}

/* x86 cvttsd2si: out-of-range / NaN -> INT_MIN (SURVEY 8a rule 4). */
static int trunc_i32_x86(double x) {
  if (!(x > -2147483649.0 && x < 2147483648.0)) return INT_MIN;
  return (int)x;
}

/* ================================================================ training */

/* stage descriptor used while scoring one layout */
typedef struct {
  const int32_t* dev;  /* devices of the block, canonical order */
  int n;
} block_t;

/* min_link_within_groups (src/cost_model.cpp:12-36) */
static double min_link_groups(const gp_cluster* c, const int32_t* dev, int n, int gsize,
                              int strided, int stride) {
  double m = K_INF;
  int groups = n / gsize;
  for (int g = 0; g < groups; ++g)
    for (int i = 0; i < gsize; ++i)
      for (int j = i + 1; j < gsize; ++j) {
        int a = strided ? dev[i * stride + g] : dev[g * gsize + i];
        int b = strided ? dev[j * stride + g] : dev[g * gsize + j];
        double l = link(c, a, b);
        if (l < m) m = l;
      }
  return m;
}

/* min_link_between (src/cost_model.cpp:38-47) */
static double min_link_between(const gp_cluster* c, block_t a, block_t b) {
  double m = K_INF;
  for (int i = 0; i < a.n; ++i)
    for (int j = 0; j < b.n; ++j) {
      double l = link(c, a.dev[i], b.dev[j]);
      if (l < m) m = l;
    }
  return m;
}

typedef struct {
  double compute, tp_comm, dp_comm;
} stage_cost_t;

/* train_stage_cost (src/cost_model.cpp:57-91) */
static stage_cost_t train_stage_cost(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                                     block_t b, int tp, int dp, int layers, int total_layers) {
  stage_cost_t sc = {0, 0, 0};
  const double tokens = w_tokens(w);
  const int type = c->device_type[b.dev[0]];
  double cap = 0;
  for (int i = 0; i < b.n; ++i) cap += c->device_flops[b.dev[i]];
  double lf = total_layers > 0 ? (double)layers / total_layers : 0;
  double need = 6.0 * w_params(w) * tokens * lf;
  sc.compute = need / (k->compute_eff[type] * cap);
  if (tp > 1 && tokens > 0) {
    double beta = min_link_groups(c, b.dev, b.n, tp, 0, 0);
    double prt = tokens / dp;
    double vol = k->tp_allreduce_coeff * layers * prt * w->hidden_dim * K_ACT_BYTES * 2.0 *
                 (tp - 1) / tp;
    sc.tp_comm = vol / beta;
  }
  if (dp > 1) {
    double beta = min_link_groups(c, b.dev, b.n, dp, 1, tp);
    double shard = w_params(w) * lf * k->grad_bytes_per_param / tp;
    double vol = 2.0 * shard * (dp - 1) / dp;
    sc.dp_comm = vol / beta;
  }
  return sc;
}

/* mem_cumsum_train (src/cost_model.cpp:198-207) */
static double mem_train_gb(const gp_workload* w, const gp_calib* k, int tp, int dp, int layers) {
  double lf = (double)layers / w->num_layers;
  double weight = w_params(w) * lf * w->bytes_per_param_train / tp;
  double tpm = w_tokens(w) / dp / w->micro_batches;
  double act = k->activation_coeff * tpm * w->hidden_dim * K_ACT_BYTES * layers / tp;
  return (weight + act) / 1e9;
}

/* allocate_layers (src/train_search.cpp:146-177). Returns 0 or GP_INVALID. */
static int allocate_layers(int L, const double* f, int S, int* layers) {
  if (S < 1 || L < S) return fail(GP_INVALID, "cannot allocate %d layers to %d stages", L, S);
  double total = 0.0;
  for (int s = 0; s < S; ++s) total += f[s];
  double rem[GP_MAX_STAGES];
  int order[GP_MAX_STAGES];
  int assigned = 0;
  for (int s = 0; s < S; ++s) {
    double share = L * f[s] / total;
    layers[s] = (int)share;
    assigned += layers[s];
    rem[s] = share - layers[s];
  }
  /* stable sort by remainder, descending (insertion sort is stable) */
  for (int s = 0; s < S; ++s) {
    int j = s;
    while (j > 0 && rem[order[j - 1]] < rem[s]) {
      order[j] = order[j - 1];
      --j;
    }
    order[j] = s;
  }
  for (int i = 0; i < L - assigned; ++i) layers[order[i % S]]++;
  for (int s = 0; s < S; ++s) {
    while (layers[s] == 0) {
      int donor = 0;
      for (int t = 1; t < S; ++t)
        if (layers[t] > layers[donor]) donor = t;
      layers[donor]--;
      layers[s]++;
    }
  }
  return 0;
}

typedef struct {
  const gp_cluster* c;
  int32_t* ordered;      /* canonical order (src/train_search.cpp:13-22) */
  int n;
  int n_runs;
  int run_start[GP_MAX_TYPES + 1];
  int run_len[GP_MAX_TYPES];
  int* cuts[GP_MAX_TYPES];   /* cut positions per run (local indices) */
  int n_cuts[GP_MAX_TYPES];
  int max_stages, max_per_run;
  int64_t cnt[GP_MAX_TYPES + 1][GP_MAX_STAGES + 2];  /* completions of runs r.. after u stages */
} layout_space_t;

static const gp_cluster* g_sort_cluster;
static int cmp_canonical(const void* pa, const void* pb) {
  int a = *(const int32_t*)pa, b = *(const int32_t*)pb;
  const gp_cluster* c = g_sort_cluster;
  if (c->device_type[a] != c->device_type[b]) return c->device_type[a] < c->device_type[b] ? -1 : 1;
  if (c->device_machine[a] != c->device_machine[b])
    return c->device_machine[a] < c->device_machine[b] ? -1 : 1;
  return a < b ? -1 : (a > b);
}

static void space_free(layout_space_t* sp) {
  free(sp->ordered);
  for (int r = 0; r < sp->n_runs; ++r) free(sp->cuts[r]);
}

/* canonical_order + build_runs + enumerate_block_lists setup
 * (src/train_search.cpp:13-50,126-142) */
static int space_build(layout_space_t* sp, const gp_cluster* c, const gp_workload* w,
                       const int32_t* ids, int n, const gp_train_opts* o) {
  memset(sp, 0, sizeof *sp);
  sp->c = c;
  sp->n = n;
  sp->ordered = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= c->n_devices) {
      free(sp->ordered);
      sp->ordered = NULL;
      return fail(GP_INVALID, "unknown device id %d", ids[i]);
    }
    sp->ordered[i] = ids[i];
  }
  g_sort_cluster = c;
  qsort(sp->ordered, (size_t)n, sizeof(int32_t), cmp_canonical);
  int dev_gran = n <= o->device_granularity_limit;
  for (int i = 0; i < n; ++i) {
    int t = c->device_type[sp->ordered[i]];
    if (i == 0 || c->device_type[sp->ordered[i - 1]] != t) {
      if (sp->n_runs == GP_MAX_TYPES) return fail(GP_INVALID, "too many runs");
      sp->run_start[sp->n_runs++] = i;
    }
  }
  sp->run_start[sp->n_runs] = n;
  for (int r = 0; r < sp->n_runs; ++r) {
    int s0 = sp->run_start[r], len = sp->run_start[r + 1] - s0;
    sp->run_len[r] = len;
    sp->cuts[r] = (int*)malloc(sizeof(int) * (size_t)(len > 0 ? len : 1));
    sp->n_cuts[r] = 0;
    for (int i = 1; i < len; ++i) {
      int edge = c->device_machine[sp->ordered[s0 + i]] != c->device_machine[sp->ordered[s0 + i - 1]];
      if (dev_gran || edge) sp->cuts[r][sp->n_cuts[r]++] = i;
    }
  }
  sp->max_per_run = o->max_stages_per_type;
  int ms = sp->n_runs * o->max_stages_per_type;
  sp->max_stages = w->num_layers < ms ? w->num_layers : ms;
  if (sp->max_stages > GP_MAX_STAGES) return fail(GP_INVALID, "max_stages exceeds GP_MAX_STAGES");
  return 0;
}

typedef struct {
  layout_space_t* sp;
  const gp_workload* w;
  const gp_calib* k;
  int window;
  int64_t rank, lo, hi;
  int64_t feasible;
  int have_best;
  double best_cost;
  int64_t best_rank;
  int n_blocks;
  int blk_start[GP_MAX_STAGES];  /* absolute offsets into ordered */
  int blk_len[GP_MAX_STAGES];
  int best_n;
  int best_start[GP_MAX_STAGES], best_len[GP_MAX_STAGES];
  int best_tp[GP_MAX_STAGES], best_dp[GP_MAX_STAGES], best_layers[GP_MAX_STAGES];
  int scoring;  /* 0: count only */
  int product;  /* enumerate_train_candidates product space instead of constrained_search */
  int64_t cand; /* product-space candidates visited */
  int err;
  double* dump; /* optional: per_step of ranks [lo, hi) (+inf: no memory-feasible option) */
} search_t;

/* max_devices_per_machine (src/train_search.cpp:74-81). A block lies inside one
 * type run of the canonical order, so equal machine ids are contiguous. */
static int max_per_machine(const gp_cluster* c, const int32_t* dev, int n) {
  int best = 0, run = 0;
  for (int i = 0; i < n; ++i) {
    run = (i > 0 && c->device_machine[dev[i]] == c->device_machine[dev[i - 1]]) ? run + 1 : 1;
    if (run > best) best = run;
  }
  return best;
}

/* train_step_cost -> train_cost_breakdown (src/cost_model.cpp:93-126) */
static double plan_step_cost(const search_t* st, const block_t* blk, int S, const int* layers,
                             const int* tps, const int* dps) {
  const gp_cluster* c = st->sp->c;
  const gp_workload* w = st->w;
  int total_layers = 0;
  for (int s = 0; s < S; ++s) total_layers += layers[s];
  double max_stage = 0, max_compute = 0;
  for (int s = 0; s < S; ++s) {
    stage_cost_t sc = train_stage_cost(c, w, st->k, blk[s], tps[s], dps[s], layers[s], total_layers);
    double tot = sc.compute + sc.tp_comm + sc.dp_comm;
    if (tot > max_stage) max_stage = tot;   /* std::max(max, v): v only if max < v */
    if (sc.compute > max_compute) max_compute = sc.compute;
  }
  double fill = 0, transfers = 0;
  const double tokens = w_tokens(w);
  if (S > 1) {
    fill = (double)(S - 1) / w->micro_batches * max_compute;
    if (tokens > 0) {
      for (int s = 0; s + 1 < S; ++s) {
        double beta = min_link_between(c, blk[s], blk[s + 1]);
        transfers += tokens * w->hidden_dim * K_ACT_BYTES / beta;
      }
    }
  }
  return max_stage + fill + transfers;  /* per_step; cost = window * per_step */
}

/* one block list of enumerate_train_candidates (src/train_search.cpp:179-216): every
 * (tp, dp) pick in odometer order (pick[0] fastest), train_plan_fits
 * (src/cost_model.cpp:232-241), train_step_cost, strict < (tests/oracles.cpp:166-174) */
static void score_layout_product(search_t* st) {
  const gp_cluster* c = st->sp->c;
  const gp_workload* w = st->w;
  const int S = st->n_blocks;
  double f[GP_MAX_STAGES];
  int layers[GP_MAX_STAGES] = {0}, tps[GP_MAX_STAGES] = {0}, dps[GP_MAX_STAGES] = {0};
  int n_opt[GP_MAX_STAGES], opt_tp[GP_MAX_STAGES][4], pick[GP_MAX_STAGES];
  block_t blk[GP_MAX_STAGES];
  for (int s = 0; s < S; ++s) {
    blk[s].dev = st->sp->ordered + st->blk_start[s];
    blk[s].n = st->blk_len[s];
    double acc = 0;
    for (int i = 0; i < blk[s].n; ++i) acc += c->device_flops[blk[s].dev[i]];
    f[s] = acc;
  }
  if (allocate_layers(w->num_layers, f, S, layers)) {
    st->err = GP_INVALID;
    return;
  }
  for (int s = 0; s < S; ++s) {  /* tp_dp_options (src/train_search.cpp:74-93) */
    int per_machine = max_per_machine(c, blk[s].dev, blk[s].n);
    static const int tp_opts[4] = {1, 2, 4, 8};
    n_opt[s] = 0;
    for (int o = 0; o < 4; ++o)
      if (tp_opts[o] <= per_machine && blk[s].n % tp_opts[o] == 0) opt_tp[s][n_opt[s]++] = tp_opts[o];
    pick[s] = 0;
  }
  for (;;) {
    int fits = 1;
    for (int s = 0; s < S; ++s) {
      tps[s] = opt_tp[s][pick[s]];
      dps[s] = blk[s].n / tps[s];
      double need_gb = mem_train_gb(w, st->k, tps[s], dps[s], layers[s]);
      for (int i = 0; i < blk[s].n; ++i)
        if (need_gb * 1e9 > c->device_hbm_cap[blk[s].dev[i]]) fits = 0;
    }
    if (fits) {
      st->feasible++;
      double cost = st->window * plan_step_cost(st, blk, S, layers, tps, dps);
      if (!st->have_best || cost < st->best_cost) {
        st->have_best = 1;
        st->best_cost = cost;
        st->best_rank = st->cand;
        st->best_n = S;
        for (int s = 0; s < S; ++s) {
          st->best_start[s] = st->blk_start[s];
          st->best_len[s] = st->blk_len[s];
          st->best_tp[s] = tps[s];
          st->best_dp[s] = dps[s];
          st->best_layers[s] = layers[s];
        }
      }
    }
    st->cand++;
    int i = 0;
    while (i < S && ++pick[i] == n_opt[i]) {
      pick[i] = 0;
      ++i;
    }
    if (i == S) break;
  }
}

/* one layout: constrained_search loop body (src/train_search.cpp:227-273) */
static void score_layout(search_t* st) {
  const gp_cluster* c = st->sp->c;
  const gp_workload* w = st->w;
  const int S = st->n_blocks;
  double f[GP_MAX_STAGES];
  int layers[GP_MAX_STAGES] = {0}, tps[GP_MAX_STAGES] = {0}, dps[GP_MAX_STAGES] = {0};
  block_t blk[GP_MAX_STAGES];
  for (int s = 0; s < S; ++s) {
    blk[s].dev = st->sp->ordered + st->blk_start[s];
    blk[s].n = st->blk_len[s];
    double acc = 0;
    for (int i = 0; i < blk[s].n; ++i) acc += c->device_flops[blk[s].dev[i]];
    f[s] = acc;
  }
  if (allocate_layers(w->num_layers, f, S, layers)) {
    st->err = GP_INVALID;
    return;
  }
  for (int s = 0; s < S; ++s) {
    double best_comm = -1;
    int per_machine = max_per_machine(c, blk[s].dev, blk[s].n);
    static const int tp_opts[4] = {1, 2, 4, 8};
    for (int o = 0; o < 4; ++o) {
      int tp = tp_opts[o];
      if (tp > per_machine || blk[s].n % tp != 0) continue;
      int dp = blk[s].n / tp;
      double need_gb = mem_train_gb(w, st->k, tp, dp, layers[s]);
      if (need_gb * 1e9 > c->device_hbm_cap[blk[s].dev[0]]) continue;
      stage_cost_t sc = train_stage_cost(c, w, st->k, blk[s], tp, dp, layers[s], w->num_layers);
      double comm = sc.tp_comm + sc.dp_comm;
      if (best_comm < 0 || comm < best_comm) {
        best_comm = comm;
        tps[s] = tp;
        dps[s] = dp;
      }
    }
    if (best_comm < 0) { /* dead layout */
      if (st->dump) st->dump[st->rank - st->lo] = HUGE_VAL;
      return;
    }
  }
  st->feasible++;
  double per_step = plan_step_cost(st, blk, S, layers, tps, dps);
  if (st->dump) st->dump[st->rank - st->lo] = per_step;
  double cost = st->window * per_step;
  if (!st->have_best || cost < st->best_cost) {
    st->have_best = 1;
    st->best_cost = cost;
    st->best_rank = st->rank;
    st->best_n = S;
    for (int s = 0; s < S; ++s) {
      st->best_start[s] = st->blk_start[s];
      st->best_len[s] = st->blk_len[s];
      st->best_tp[s] = tps[s];
      st->best_dp[s] = dps[s];
      st->best_layers[s] = layers[s];
    }
  }
}

static void visit_leaf(search_t* st) {
  if (st->scoring && st->rank >= st->lo && st->rank < st->hi && !st->err) {
    if (st->product) score_layout_product(st);
    else score_layout(st);
  }
  st->rank++;
}

static void recurse_runs(search_t* st, int r, int used);

/* run_compositions (src/train_search.cpp:53-72): choose k-1 cuts in lexicographic order */
static void recurse_cuts(search_t* st, int r, int used, int k, int chosen, int next_cut, int prev) {
  layout_space_t* sp = st->sp;
  int base = sp->run_start[r];
  if (chosen == k - 1) {
    st->blk_start[used + chosen] = base + prev;
    st->blk_len[used + chosen] = sp->run_len[r] - prev;
    st->n_blocks = used + k;
    /* skip whole subtrees outside [lo, hi): their size is cnt[r+1][used+k] */
    int64_t size = sp->cnt[r + 1][used + k];
    if (st->rank + size <= st->lo || st->rank >= st->hi) {
      st->rank += size;
      return;
    }
    recurse_runs(st, r + 1, used + k);
    return;
  }
  int remaining = k - 1 - chosen;
  for (int ci = next_cut; ci + remaining <= sp->n_cuts[r]; ++ci) {
    int cut = sp->cuts[r][ci];
    st->blk_start[used + chosen] = base + prev;
    st->blk_len[used + chosen] = cut - prev;
    recurse_cuts(st, r, used, k, chosen + 1, ci + 1, cut);
  }
}

/* Enumerator::recurse (src/train_search.cpp:95-124) */
static void recurse_runs(search_t* st, int r, int used) {
  layout_space_t* sp = st->sp;
  if (r == sp->n_runs) {
    visit_leaf(st);
    return;
  }
  int remaining_runs = sp->n_runs - r - 1;
  int kmax = sp->max_per_run < sp->run_len[r] ? sp->max_per_run : sp->run_len[r];
  for (int k = 1; k <= kmax; ++k) {
    if (used + k + remaining_runs > sp->max_stages) break;
    recurse_cuts(st, r, used, k, 0, 0, 0);
  }
}

/* Layout count without enumeration: cnt[r][u] recurrence. */
static int64_t binom(int n, int k) {
  if (k < 0 || k > n) return 0;
  int64_t v = 1;
  for (int i = 1; i <= k; ++i) v = v * (n - k + i) / i;
  return v;
}

static int64_t count_layouts(layout_space_t* sp) {
  if (sp->max_stages < sp->n_runs) return 0;
  memset(sp->cnt, 0, sizeof sp->cnt);
  for (int u = 0; u <= sp->max_stages; ++u) sp->cnt[sp->n_runs][u] = 1;
  for (int r = sp->n_runs - 1; r >= 0; --r) {
    int remaining_runs = sp->n_runs - r - 1;
    for (int u = 0; u <= sp->max_stages; ++u) {
      int64_t acc = 0;
      int kmax = sp->max_per_run < sp->run_len[r] ? sp->max_per_run : sp->run_len[r];
      for (int k = 1; k <= kmax; ++k) {
        if (u + k + remaining_runs > sp->max_stages) break;
        acc += binom(sp->n_cuts[r], k - 1) * sp->cnt[r + 1][u + k];
      }
      sp->cnt[r][u] = acc;
    }
  }
  return sp->cnt[0][0];
}

int or_train_space(const gp_cluster* c, const gp_workload* w, const int32_t* ids, int32_t n,
                   const gp_train_opts* opts, int64_t* layouts) {
  layout_space_t sp;
  int rc = space_build(&sp, c, w, ids, n, opts);
  if (rc) return rc;
  *layouts = count_layouts(&sp);
  space_free(&sp);
  return GP_OK;
}

/* constrained_search (src/train_search.cpp:218-275), restricted to ranks [lo, hi). */
static int constrained_search_impl(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                                   const int32_t* ids, int32_t n, int32_t window,
                                   const gp_train_opts* opts, int64_t lo, int64_t hi,
                                   gp_train_result* out, int32_t* stage_devices, double* dump) {
  memset(out, 0, sizeof *out);
  if (n <= 0) return fail(GP_INVALID, "constrained_search requires a non-empty train set");
  layout_space_t sp;
  int rc = space_build(&sp, c, w, ids, n, opts);
  if (rc) return rc;
  int64_t total = count_layouts(&sp);
  if (hi < 0 || hi > total) hi = total;
  if (lo < 0) lo = 0;
  search_t st;
  memset(&st, 0, sizeof st);
  st.sp = &sp;
  st.w = w;
  st.k = k;
  st.window = window;
  st.lo = lo;
  st.hi = hi;
  st.scoring = 1;
  st.dump = dump;
  if (sp.max_stages >= sp.n_runs && lo < hi) recurse_runs(&st, 0, 0);
  out->layouts = hi > lo ? hi - lo : 0;
  out->feasible = st.feasible;
  if (st.err) {
    space_free(&sp);
    return st.err;
  }
  if (st.have_best) {
    out->found = 1;
    out->cost = st.best_cost;
    out->rank = st.best_rank;
    out->n_stages = st.best_n;
    int off = 0;
    for (int s = 0; s < st.best_n; ++s) {
      out->stage[s].first = off;
      out->stage[s].count = st.best_len[s];
      out->stage[s].tp = st.best_tp[s];
      out->stage[s].dp = st.best_dp[s];
      out->stage[s].layers = st.best_layers[s];
      for (int i = 0; i < st.best_len[s]; ++i)
        stage_devices[off++] = sp.ordered[st.best_start[s] + i];
    }
  }
  space_free(&sp);
  return GP_OK;
}

int or_constrained_search(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                          const int32_t* ids, int32_t n, int32_t window, const gp_train_opts* opts,
                          int64_t lo, int64_t hi, gp_train_result* out, int32_t* stage_devices) {
  return constrained_search_impl(c, w, k, ids, n, window, opts, lo, hi, out, stage_devices, NULL);
}

/* per_step (train_cost_breakdown(...).per_step, src/cost_model.cpp:123) of every layout of
 * ranks [lo, hi) in enumeration order, +inf for layouts without a memory-feasible option
 * (src/train_search.cpp:260-266). hi must not exceed the space size. */
int or_layout_costs(const gp_cluster* c, const gp_workload* w, const gp_calib* k, const int32_t* ids,
                    int32_t n, const gp_train_opts* opts, int64_t lo, int64_t hi, double* per_step) {
  gp_train_result res;
  int32_t* devs = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int rc = constrained_search_impl(c, w, k, ids, n, 1, opts, lo, hi, &res, devs, per_step);
  free(devs);
  return rc;
}

int or_train_candidates_search(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                               const int32_t* ids, int32_t n, int32_t window, gp_train_result* out,
                               int32_t* stage_devices) {
  memset(out, 0, sizeof *out);
  if (n <= 0) return fail(GP_INVALID, "enumerate_train_candidates requires a non-empty train set");
  gp_train_opts opts = {4, 16};  /* TrainSearchOptions defaults */
  layout_space_t sp;
  int rc = space_build(&sp, c, w, ids, n, &opts);
  if (rc) return rc;
  search_t st;
  memset(&st, 0, sizeof st);
  st.sp = &sp;
  st.w = w;
  st.k = k;
  st.window = window;
  st.lo = 0;
  st.hi = INT64_MAX;
  st.scoring = 1;
  st.product = 1;
  count_layouts(&sp);  /* the enumeration's subtree sizes */
  if (sp.max_stages >= sp.n_runs) recurse_runs(&st, 0, 0);
  out->layouts = st.cand;
  out->feasible = st.feasible;
  if (st.err) {
    space_free(&sp);
    return st.err;
  }
  if (st.have_best) {
    out->found = 1;
    out->cost = st.best_cost;
    out->rank = st.best_rank;
    out->n_stages = st.best_n;
    int off = 0;
    for (int s = 0; s < st.best_n; ++s) {
      out->stage[s].first = off;
      out->stage[s].count = st.best_len[s];
      out->stage[s].tp = st.best_tp[s];
      out->stage[s].dp = st.best_dp[s];
      out->stage[s].layers = st.best_layers[s];
      for (int i = 0; i < st.best_len[s]; ++i) stage_devices[off++] = sp.ordered[st.best_start[s] + i];
    }
  }
  space_free(&sp);
  return GP_OK;
}

/* ================================================================ rollout */

int or_rollout_capacities(const gp_cluster* c, const int32_t* ids, int32_t n, int32_t* caps) {
  /* src/rollout_milp.cpp:30-37 */
  for (int t = 0; t < c->n_types; ++t) caps[t] = 0;
  for (int i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= c->n_devices) return fail(GP_INVALID, "unknown device id %d", ids[i]);
    caps[c->device_type[ids[i]]]++;
  }
  return GP_OK;
}

static int config_type(const gp_config* cfg, int n_types) {
  for (int t = 0; t < n_types; ++t)
    if (cfg->type_counts[t] > 0) return t;
  return -1;
}

/* layers_for_stage (src/cost_model.cpp:51-55) */
static int layers_for_stage(int layers, int stages, int index) {
  return layers / stages + (index < layers % stages ? 1 : 0);
}

/* replica_concurrency (src/cost_model.cpp:128-148) */
static int replica_concurrency(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                               const gp_config* cfg) {
  int type = config_type(cfg, c->n_types);
  if (type < 0) return 0;
  int S = cfg->n_stages;
  int best = k->max_concurrency;
  for (int s = 0; s < S; ++s) {
    int layers = layers_for_stage(w->num_layers, S, s);
    int tp = cfg->tp[s];
    double lf = (double)layers / w->num_layers;
    double weight = w_params(w) * lf * w->bytes_per_param_infer / tp;
    double free_b = c->type_hbm_cap[type] - weight;
    if (free_b < 0) return 0;
    double kv = w_kv_bytes_per_token(w) * w_mean_total_len(w) * lf / tp;
    if (kv > 0) {
      int v = trunc_i32_x86(free_b / kv);
      if (v < best) best = v;
    }
  }
  return best > 0 ? best : 0;
}

/* replica_rate_at (src/cost_model.cpp:150-165) */
static double replica_rate_at(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                              const gp_config* cfg, double conc) {
  double agg_bw = 0, agg_flops = 0;
  for (int t = 0; t < c->n_types; ++t) {
    if (cfg->type_counts[t] == 0) continue;
    agg_bw += cfg->type_counts[t] * c->type_hbm_bw[t] * k->io_eff[t];
    agg_flops += cfg->type_counts[t] * c->type_flops[t] * k->compute_eff[t];
  }
  double io = conc * agg_bw / w_model_bytes_infer(w);
  double comp = agg_flops / (2.0 * w_params(w));
  double pen = 1.0 + k->stage_latency_penalty * (cfg->n_stages - 1);
  double m = comp < io ? comp : io;
  return m / pen;
}

static void tp_multisets(int stages, int max_tp, int* acc, int depth, gp_config* tmpl,
                         int (*emit)(void*, const int*), void* ud) {
  if (depth == stages) {
    emit(ud, acc);
    return;
  }
  static const int tps[4] = {8, 4, 2, 1};
  for (int i = 0; i < 4; ++i) {
    if (tps[i] > max_tp) continue;
    acc[depth] = tps[i];
    tp_multisets(stages, tps[i], acc, depth + 1, tmpl, emit, ud);
  }
}

typedef struct {
  const gp_cluster* c;
  const gp_workload* w;
  const gp_calib* k;
  int type, stages;
  const int* avail;
  gp_config* out;
  int cap, n, overflow;
} cfg_emit_t;

static int emit_cfg(void* ud, const int* tps) {
  cfg_emit_t* e = (cfg_emit_t*)ud;
  for (int s = 0; s < e->stages; ++s)
    if (tps[s] > e->avail[s]) return 0;
  gp_config cfg;
  memset(&cfg, 0, sizeof cfg);
  for (int s = 0; s < e->stages; ++s) {
    cfg.type_counts[e->type] += tps[s];
    cfg.tp[s] = tps[s];
  }
  cfg.n_stages = e->stages;
  int conc = replica_concurrency(e->c, e->w, e->k, &cfg);
  if (conc < 1) return 0;
  cfg.throughput = replica_rate_at(e->c, e->w, e->k, &cfg, (double)conc);
  if (e->n < e->cap) e->out[e->n] = cfg;
  else e->overflow = 1;
  e->n++;
  return 0;
}

static int cmp_desc_int(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return (x < y) - (x > y);
}

/* enumerate_configs (src/rollout_milp.cpp:39-89) */
int or_enumerate_configs(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                         const int32_t* ids, int32_t n, const gp_rollout_opts* opts,
                         gp_config* out, int32_t cap, int32_t* n_out) {
  if (n <= 0) return fail(GP_INVALID, "enumerate_configs requires a non-empty rollout set");
  if (opts->max_stages > GP_MAX_ROLLOUT_STAGES)
    return fail(GP_INVALID, "max_stages exceeds GP_MAX_ROLLOUT_STAGES");
  int* per_machine = (int*)calloc((size_t)c->n_machines, sizeof(int));
  int* avail = (int*)malloc(sizeof(int) * (size_t)c->n_machines);
  cfg_emit_t e = {c, w, k, 0, 0, avail, out, cap, 0, 0};
  for (int i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= c->n_devices) {
      free(per_machine);
      free(avail);
      return fail(GP_INVALID, "unknown device id %d", ids[i]);
    }
  for (int t = 0; t < c->n_types; ++t) {
    memset(per_machine, 0, sizeof(int) * (size_t)c->n_machines);
    for (int i = 0; i < n; ++i)
      if (c->device_type[ids[i]] == t) per_machine[c->device_machine[ids[i]]]++;
    int na = 0;
    for (int m = 0; m < c->n_machines; ++m)
      if (per_machine[m] > 0) avail[na++] = per_machine[m];
    if (na == 0) continue;
    qsort(avail, (size_t)na, sizeof(int), cmp_desc_int);
    int ms = opts->max_stages;
    if (na < ms) ms = na;
    if (w->num_layers < ms) ms = w->num_layers;
    e.type = t;
    for (int s = 1; s <= ms; ++s) {
      int acc[GP_MAX_ROLLOUT_STAGES];
      e.stages = s;
      tp_multisets(s, 8, acc, 0, NULL, emit_cfg, &e);
    }
  }
  free(per_machine);
  free(avail);
  *n_out = e.n;
  if (e.overflow) return fail(GP_CAPACITY, "config buffer too small (%d needed)", e.n);
  return GP_OK;
}

/* solve_milp (src/rollout_milp.cpp:91-171) */
int or_solve_milp(const gp_config* cfg, int32_t nc, const int32_t* caps, int32_t dims, double B,
                  double len, gp_rollout_result* out, gp_rollout_entry* entries) {
  memset(out, 0, sizeof *out);
  out->total_rollouts = B;
  if (B <= 0) return GP_OK;
  if (nc == 0) return fail(GP_INFEASIBLE, "no replica configuration available");
  int64_t stride[GP_MAX_TYPES];
  int64_t states = 1;
  for (int t = 0; t < dims; ++t) {
    stride[t] = states;
    states *= caps[t] + 1;
    if (states > 50000000) return fail(GP_INVALID, "capacity lattice too large for the exact solver");
  }
  out->states = states;
  double* best = (double*)malloc(sizeof(double) * (size_t)states);
  int* choice = (int*)malloc(sizeof(int) * (size_t)states);
  for (int64_t s = 0; s < states; ++s) {
    best[s] = 0.0;
    choice[s] = -1;
  }
  int sv[GP_MAX_TYPES];
  for (int64_t s = 0; s < states; ++s) {
    int64_t rem = s;
    for (int t = dims - 1; t >= 0; --t) {
      sv[t] = (int)(rem / stride[t]);
      rem %= stride[t];
    }
    for (int ci = 0; ci < nc; ++ci) {
      int64_t prev = s;
      int ok = 1;
      for (int t = 0; t < dims; ++t) {
        int need = cfg[ci].type_counts[t];
        if (sv[t] < need) {
          ok = 0;
          break;
        }
        prev -= (int64_t)need * stride[t];
      }
      if (!ok) continue;
      double cand = best[prev] + cfg[ci].throughput;
      if (cand > best[s]) {
        best[s] = cand;
        choice[s] = ci;
      }
    }
  }
  int64_t full = states - 1;
  double agg = best[full];
  out->aggregate = agg;
  if (agg <= 0) {
    free(best);
    free(choice);
    return fail(GP_INFEASIBLE, "rollout capacity cannot host any replica");
  }
  int* counts = (int*)calloc((size_t)nc, sizeof(int));
  int64_t cur = full;
  while (choice[cur] >= 0) {
    int ci = choice[cur];
    counts[ci]++;
    for (int t = 0; t < dims; ++t) cur -= (int64_t)cfg[ci].type_counts[t] * stride[t];
  }
  out->makespan = B * len / agg;
  int ne = 0;
  for (int ci = 0; ci < nc; ++ci) {
    if (counts[ci] == 0) continue;
    entries[ne].config = ci;
    entries[ne].replicas = counts[ci];
    entries[ne].workload = B * counts[ci] * cfg[ci].throughput / agg;
    ne++;
  }
  out->n_entries = ne;
  free(counts);
  free(best);
  free(choice);
  return GP_OK;
}

/* weight_sync_cost (src/cost_model.cpp:174-196) */
int or_weight_sync_cost(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                        const int32_t* train, int32_t nt, const int32_t* roll, int32_t nr,
                        const int32_t* etype, const int32_t* erep, int32_t ne, int32_t window,
                        double* out) {
  double bottleneck = K_INF;
  for (int e = 0; e < ne; ++e) {
    if (erep[e] < 1) continue;
    int type = etype[e];
    double best = 0;
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j < nr; ++j) {
        if (c->device_type[roll[j]] != type) continue;
        double l = link(c, train[i], roll[j]);
        if (best < l) best = l;
      }
    if (best > 0 && best < bottleneck) bottleneck = best;
  }
  double transfer = 0;
  if (bottleneck < K_INF && w_model_bytes_infer(w) > 0) transfer = w_model_bytes_infer(w) / bottleneck;
  *out = window * transfer + k->sync_latency_s;
  return GP_OK;
}

/* ====================================================== exhaustive (tests/oracles.cpp) */

typedef struct {
  const gp_config* cfg;
  int nc, dims;
  int caps[GP_MAX_TYPES];
  double B, len;
  int feasible;
  double theta;
  int32_t* best;
  int cur[512];
  int64_t vectors;
} brute_t;

/* enumerate_all's Rec::go (tests/oracles.cpp:34-66) */
static void brute_go(brute_t* b, int idx, double agg) {
  if (idx == b->nc) {
    b->vectors++;
    if (agg <= 0) return;
    double theta = b->B * b->len / agg;
    if (!b->feasible || theta < b->theta - 1e-15) {
      b->feasible = 1;
      b->theta = theta;
      for (int i = 0; i < b->nc; ++i) b->best[i] = b->cur[i];
    }
    return;
  }
  const int32_t* v = b->cfg[idx].type_counts;
  int bound = INT32_MAX, uses = 0;
  for (int t = 0; t < b->dims; ++t)
    if (v[t] > 0) {
      uses = 1;
      int q = b->caps[t] / v[t];
      if (q < bound) bound = q;
    }
  if (!uses) bound = 0;
  for (int y = 0; y <= bound; ++y) {
    b->cur[idx] = y;
    for (int t = 0; t < b->dims; ++t) b->caps[t] -= y * v[t];
    brute_go(b, idx + 1, agg + y * b->cfg[idx].throughput);
    for (int t = 0; t < b->dims; ++t) b->caps[t] += y * v[t];
  }
}

int or_brute_milp(const gp_config* configs, int32_t n_configs, const int32_t* caps, int32_t dims,
                  double total_rollouts, double mean_len, int32_t* feasible, double* theta,
                  int32_t* counts, int64_t* vectors) {
  if (n_configs > 512 || dims > GP_MAX_TYPES) return fail(GP_INVALID, "brute_milp instance too large");
  for (int i = 0; i < n_configs; ++i) counts[i] = 0;
  *vectors = 0;
  if (total_rollouts <= 0) {
    *feasible = 1;
    *theta = 0;
    return GP_OK;
  }
  brute_t b;
  memset(&b, 0, sizeof b);
  b.cfg = configs;
  b.nc = n_configs;
  b.dims = dims;
  for (int t = 0; t < dims; ++t) b.caps[t] = caps[t];
  b.B = total_rollouts;
  b.len = mean_len;
  b.best = counts;
  brute_go(&b, 0, 0.0);
  *feasible = b.feasible;
  *theta = b.theta;
  *vectors = b.vectors;
  return GP_OK;
}

int or_exhaustive_optimum(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                          int32_t window, gp_exhaustive_result* out, int32_t* train_ids) {
  memset(out, 0, sizeof *out);
  const int n = c->n_devices;
  if (n < 2 || n > 30) return fail(GP_INVALID, "exhaustive optimum needs 2 <= devices <= 30");
  const double total_rollouts = (double)w->batch_rollouts * window;
  int have = 0, have_c = 0;
  double best = 0, best_c = 0;
  uint32_t best_mask = 0, best_mask_c = 0;
  int32_t train[32], roll[32], sdev[32], caps[GP_MAX_TYPES], counts[512], et[512], er[512];
  gp_config cfg[512];
  for (uint32_t mask = 1; mask + 1 < (1u << n); ++mask) {
    int nt = 0, nr = 0;
    for (int d = 0; d < n; ++d) {
      if (mask & (1u << d)) train[nt++] = d;
      else roll[nr++] = d;
    }
    out->partitions++;
    gp_train_result tr;
    int rc = or_train_candidates_search(c, w, k, train, nt, window, &tr, sdev);
    if (rc) return rc;
    out->train_candidates += tr.layouts;
    if (!tr.found) continue;
    const double c_train = tr.cost;
    gp_rollout_opts ro = {4};
    int32_t ncfg = 0;
    rc = or_enumerate_configs(c, w, k, roll, nr, &ro, cfg, 512, &ncfg);
    if (rc) return rc;
    if (ncfg == 0) continue;
    rc = or_rollout_capacities(c, roll, nr, caps);
    if (rc) return rc;
    int32_t feas;
    double theta;
    int64_t vec;
    rc = or_brute_milp(cfg, ncfg, caps, c->n_types, total_rollouts, w->mean_len, &feas, &theta, counts, &vec);
    if (rc) return rc;
    out->replica_vectors += vec;
    if (!feas) continue;
    int ne = 0;
    for (int i = 0; i < ncfg; ++i)
      if (counts[i] > 0) {
        int t = 0;
        while (t < c->n_types && cfg[i].type_counts[t] == 0) ++t;
        et[ne] = t;
        er[ne] = counts[i];
        ++ne;
      }
    double update;
    rc = or_weight_sync_cost(c, w, k, train, nt, roll, nr, et, er, ne, window, &update);
    if (rc) return rc;
    const double c_infer = theta + w->reward_cost_const + update;
    const double objective = c_train < c_infer ? c_infer : c_train;  /* std::max */
    if (!have || objective < best) {
      have = 1;
      best = objective;
      best_mask = mask;
    }
    if (c_infer >= c_train && (!have_c || objective < best_c)) {
      have_c = 1;
      best_c = objective;
      best_mask_c = mask;
    }
  }
  const uint32_t m = have_c ? best_mask_c : best_mask;
  out->feasible = have_c || have;
  out->objective = have_c ? best_c : best;
  if (out->feasible)
    for (int d = 0; d < n; ++d)
      if (m & (1u << d)) train_ids[out->n_train++] = d;
  return GP_OK;
}

/* ============================================ table-memoised constrained_search
 * TEST INFRASTRUCTURE: the same restatement as or_constrained_search above, with the
 * pure sub-results memoised so a full C5 train set (2.4e9 layouts) finishes on the host
 * cores in minutes. Nothing is re-associated: each memo holds the value the plain
 * restatement computes —
 *   * min_link_within_groups per (block, tp option) and min_link_between per adjacent
 *     block pair (src/cost_model.cpp:12-47; exact minima over the device-pair matrix);
 *   * the per-stage option pick + train_stage_cost per (block, layer count)
 *     (src/train_search.cpp:241-265, src/cost_model.cpp:57-91, total_layers == L);
 *   * the block FLOPS left fold (src/train_search.cpp:229-232).
 * Per layout it runs allocate_layers (src/train_search.cpp:146-177) and
 * train_cost_breakdown's max / fill-drain / transfer fold (src/cost_model.cpp:93-126)
 * exactly as above, and keeps the first rank of minimal window*per_step per window.
 * Independent of every engine shortcut (constant allocation totals, promotion/donation
 * tables, machine-pair link tables, near-minimum summaries). Rank ranges are split over
 * pthreads; per-window (cost, rank) minima merge lexicographically. */
#include <pthread.h>
#include <stdatomic.h>

typedef struct {
  int start, n, type, per_machine;
  double f, cap0;
  double beta_tp[4], beta_dp[4];
  double* tot;       /* [L] stage total of the comm-minimal memory-feasible option */
  double* comp;      /* [L] compute */
  signed char* ok;   /* [L] 0: no memory-feasible option */
} tab_block_t;

typedef struct {
  layout_space_t* sp;
  const gp_workload* w;
  const gp_calib* k;
  int L;
  int n_pos[GP_MAX_TYPES];          /* cut positions incl. 0 and len: nc + 2 */
  int* pos[GP_MAX_TYPES];
  int blk_off[GP_MAX_TYPES];
  tab_block_t* blk;                 /* per run: [i][j] for 0 <= i < j < n_pos */
  double* tin[GP_MAX_TYPES];        /* [i][j][l]: beta between (i,j) and (j,l) of run r */
  double* tx[GP_MAX_TYPES];         /* [i][l]: beta between (i, last) of run r and (0, l) of r+1 */
  int n_windows;
  const int32_t* windows;
} tab_t;

static int tab_bid(const tab_t* t, int r, int i, int j) {
  return t->blk_off[r] + i * t->n_pos[r] + j;
}

static void tab_free(tab_t* t) {
  for (int r = 0; r < t->sp->n_runs; ++r) {
    free(t->pos[r]);
    free(t->tin[r]);
    free(t->tx[r]);
  }
  if (t->blk) {
    int nb = t->blk_off[t->sp->n_runs];
    for (int b = 0; b < nb; ++b) {
      free(t->blk[b].tot);
      free(t->blk[b].comp);
      free(t->blk[b].ok);
    }
  }
  free(t->blk);
}

static void tab_block_fill(tab_t* t, tab_block_t* b) {
  const gp_cluster* c = t->sp->c;
  const gp_workload* w = t->w;
  const gp_calib* k = t->k;
  const int32_t* dev = t->sp->ordered + b->start;
  const int L = t->L;
  double f = 0;
  for (int i = 0; i < b->n; ++i) f += c->device_flops[dev[i]];
  b->f = f;
  b->type = c->device_type[dev[0]];
  b->cap0 = c->device_hbm_cap[dev[0]];
  b->per_machine = max_per_machine(c, dev, b->n);
  static const int tp_opts[4] = {1, 2, 4, 8};
  for (int o = 0; o < 4; ++o) {
    b->beta_tp[o] = b->beta_dp[o] = K_INF;
    int tp = tp_opts[o];
    if (tp > b->per_machine || b->n % tp != 0) continue;
    int dp = b->n / tp;
    if (tp > 1) b->beta_tp[o] = min_link_groups(c, dev, b->n, tp, 0, 0);
    if (dp > 1) b->beta_dp[o] = min_link_groups(c, dev, b->n, dp, 1, tp);
  }
  b->tot = (double*)malloc(sizeof(double) * (size_t)L);
  b->comp = (double*)malloc(sizeof(double) * (size_t)L);
  b->ok = (signed char*)malloc((size_t)L);
  const double tokens = w_tokens(w);
  for (int layers = 1; layers <= L; ++layers) {
    double best_comm = -1, best_tot = 0, best_comp = 0;
    for (int o = 0; o < 4; ++o) {
      int tp = tp_opts[o];
      if (tp > b->per_machine || b->n % tp != 0) continue;
      int dp = b->n / tp;
      double need_gb = mem_train_gb(w, k, tp, dp, layers);
      if (need_gb * 1e9 > b->cap0) continue;
      /* train_stage_cost (as above) with the memoised betas; total_layers == L */
      stage_cost_t sc = {0, 0, 0};
      double lf = (double)layers / L;
      double need = 6.0 * w_params(w) * tokens * lf;
      sc.compute = need / (k->compute_eff[b->type] * f);
      if (tp > 1 && tokens > 0) {
        double prt = tokens / dp;
        double vol = k->tp_allreduce_coeff * layers * prt * w->hidden_dim * K_ACT_BYTES * 2.0 *
                     (tp - 1) / tp;
        sc.tp_comm = vol / b->beta_tp[o];
      }
      if (dp > 1) {
        double shard = w_params(w) * lf * k->grad_bytes_per_param / tp;
        double vol = 2.0 * shard * (dp - 1) / dp;
        sc.dp_comm = vol / b->beta_dp[o];
      }
      double comm = sc.tp_comm + sc.dp_comm;
      if (best_comm < 0 || comm < best_comm) {
        best_comm = comm;
        best_tot = sc.compute + sc.tp_comm + sc.dp_comm;  /* TrainStageCost::total() */
        best_comp = sc.compute;
      }
    }
    b->ok[layers - 1] = best_comm >= 0;
    b->tot[layers - 1] = best_tot;
    b->comp[layers - 1] = best_comp;
  }
}

static double tab_between(const tab_t* t, int s0, int n0, int s1, int n1) {
  block_t a = {t->sp->ordered + s0, n0}, b = {t->sp->ordered + s1, n1};
  return min_link_between(t->sp->c, a, b);
}

static int tab_build(tab_t* t, layout_space_t* sp, const gp_workload* w, const gp_calib* k) {
  memset(t, 0, sizeof *t);
  t->sp = sp;
  t->w = w;
  t->k = k;
  t->L = w->num_layers;
  int nb = 0;
  for (int r = 0; r < sp->n_runs; ++r) {
    int np = sp->n_cuts[r] + 2;
    t->n_pos[r] = np;
    t->pos[r] = (int*)malloc(sizeof(int) * (size_t)np);
    t->pos[r][0] = 0;
    for (int i = 0; i < sp->n_cuts[r]; ++i) t->pos[r][i + 1] = sp->cuts[r][i];
    t->pos[r][np - 1] = sp->run_len[r];
    t->blk_off[r] = nb;
    nb += np * np;
  }
  t->blk_off[sp->n_runs] = nb;
  t->blk = (tab_block_t*)calloc((size_t)nb, sizeof(tab_block_t));
  for (int r = 0; r < sp->n_runs; ++r) {
    int np = t->n_pos[r];
    for (int i = 0; i < np; ++i)
      for (int j = i + 1; j < np; ++j) {
        tab_block_t* b = &t->blk[tab_bid(t, r, i, j)];
        b->start = sp->run_start[r] + t->pos[r][i];
        b->n = t->pos[r][j] - t->pos[r][i];
        tab_block_fill(t, b);
      }
    t->tin[r] = (double*)malloc(sizeof(double) * (size_t)np * np * np);
    for (int i = 0; i < np; ++i)
      for (int j = i + 1; j < np; ++j)
        for (int l = j + 1; l < np; ++l) {
          const tab_block_t* a = &t->blk[tab_bid(t, r, i, j)];
          const tab_block_t* b = &t->blk[tab_bid(t, r, j, l)];
          t->tin[r][((size_t)i * np + j) * np + l] = tab_between(t, a->start, a->n, b->start, b->n);
        }
    if (r + 1 < sp->n_runs) {
      int np2 = sp->n_cuts[r + 1] + 2;
      t->tx[r] = (double*)malloc(sizeof(double) * (size_t)np * np2);
      for (int i = 0; i + 1 < np; ++i)
        for (int l = 1; l < np2; ++l) {
          int s0 = sp->run_start[r] + t->pos[r][i], n0 = sp->run_len[r] - t->pos[r][i];
          int s1 = sp->run_start[r + 1], n1 = t->pos[r + 1][l];
          t->tx[r][(size_t)i * np2 + l] = tab_between(t, s0, n0, s1, n1);
        }
    }
  }
  return 0;
}

#define TAB_MAX_WINDOWS 8
typedef struct {
  const tab_t* t;
  int64_t rank, lo, hi, feasible;
  int S;
  int run_of[GP_MAX_STAGES], pi[GP_MAX_STAGES], pj[GP_MAX_STAGES];
  int have[TAB_MAX_WINDOWS];
  double best_cost[TAB_MAX_WINDOWS];
  int64_t best_rank[TAB_MAX_WINDOWS];
  double* dump;  /* per_step of ranks [lo, hi) (+inf: no memory-feasible option) */
} tab_search_t;

static void tab_score(tab_search_t* s) {
  const tab_t* t = s->t;
  const gp_workload* w = t->w;
  const int S = s->S, L = t->L;
  double f[GP_MAX_STAGES];
  int layers[GP_MAX_STAGES];
  const tab_block_t* blk[GP_MAX_STAGES];
  for (int q = 0; q < S; ++q) {
    blk[q] = &t->blk[tab_bid(t, s->run_of[q], s->pi[q], s->pj[q])];
    f[q] = blk[q]->f;
  }
  allocate_layers(L, f, S, layers);
  double max_stage = 0, max_compute = 0;
  for (int q = 0; q < S; ++q) {
    if (!blk[q]->ok[layers[q] - 1]) {
      if (s->dump) s->dump[s->rank - s->lo] = HUGE_VAL;
      return;
    }
    double tot = blk[q]->tot[layers[q] - 1], cmp = blk[q]->comp[layers[q] - 1];
    if (tot > max_stage) max_stage = tot;
    if (cmp > max_compute) max_compute = cmp;
  }
  double fill = 0, transfers = 0;
  const double tokens = w_tokens(w);
  if (S > 1) {
    fill = (double)(S - 1) / w->micro_batches * max_compute;
    if (tokens > 0) {
      for (int q = 0; q + 1 < S; ++q) {
        double beta;
        int r = s->run_of[q];
        if (s->run_of[q + 1] == r) {
          int np = t->n_pos[r];
          beta = t->tin[r][((size_t)s->pi[q] * np + s->pj[q]) * np + s->pj[q + 1]];
        } else {
          beta = t->tx[r][(size_t)s->pi[q] * t->n_pos[r + 1] + s->pj[q + 1]];
        }
        transfers += tokens * w->hidden_dim * K_ACT_BYTES / beta;
      }
    }
  }
  double per_step = max_stage + fill + transfers;
  s->feasible++;
  if (s->dump) s->dump[s->rank - s->lo] = per_step;
  for (int i = 0; i < t->n_windows; ++i) {
    double cost = t->windows[i] * per_step;
    if (!s->have[i] || cost < s->best_cost[i]) {
      s->have[i] = 1;
      s->best_cost[i] = cost;
      s->best_rank[i] = s->rank;
    }
  }
}

static void tab_runs(tab_search_t* s, int r, int used);

static void tab_cuts(tab_search_t* s, int r, int used, int k, int chosen, int next, int prev_i) {
  const layout_space_t* sp = s->t->sp;
  if (chosen == k - 1) {
    s->run_of[used + chosen] = r;
    s->pi[used + chosen] = prev_i;
    s->pj[used + chosen] = sp->n_cuts[r] + 1;
    int64_t size = sp->cnt[r + 1][used + k];
    if (s->rank + size <= s->lo || s->rank >= s->hi) {
      s->rank += size;
      return;
    }
    tab_runs(s, r + 1, used + k);
    return;
  }
  int remaining = k - 1 - chosen;
  for (int ci = next; ci + remaining <= sp->n_cuts[r]; ++ci) {
    s->run_of[used + chosen] = r;
    s->pi[used + chosen] = prev_i;
    s->pj[used + chosen] = ci + 1;
    tab_cuts(s, r, used, k, chosen + 1, ci + 1, ci + 1);
  }
}

static void tab_runs(tab_search_t* s, int r, int used) {
  const layout_space_t* sp = s->t->sp;
  if (r == sp->n_runs) {
    if (s->rank >= s->lo && s->rank < s->hi) {
      s->S = used;
      tab_score(s);
    }
    s->rank++;
    return;
  }
  int remaining_runs = sp->n_runs - r - 1;
  int kmax = sp->max_per_run < sp->run_len[r] ? sp->max_per_run : sp->run_len[r];
  for (int k = 1; k <= kmax; ++k) {
    if (used + k + remaining_runs > sp->max_stages) break;
    tab_cuts(s, r, used, k, 0, 0, 0);
  }
}

typedef struct {
  const tab_t* t;
  int64_t lo, hi, chunk;
  atomic_llong next;
  pthread_mutex_t mu;
  tab_search_t acc;
  double* dump;
} tab_job_t;

static void tab_merge(tab_search_t* into, const tab_search_t* s, int n_windows) {
  into->feasible += s->feasible;
  for (int i = 0; i < n_windows; ++i) {
    if (!s->have[i]) continue;
    if (!into->have[i] || s->best_cost[i] < into->best_cost[i] ||
        (s->best_cost[i] == into->best_cost[i] && s->best_rank[i] < into->best_rank[i])) {
      into->have[i] = 1;
      into->best_cost[i] = s->best_cost[i];
      into->best_rank[i] = s->best_rank[i];
    }
  }
}

static void* tab_worker(void* arg) {
  tab_job_t* j = (tab_job_t*)arg;
  tab_search_t loc;
  memset(&loc, 0, sizeof loc);
  for (;;) {
    int64_t a = atomic_fetch_add(&j->next, j->chunk);
    if (a >= j->hi) break;
    int64_t b = a + j->chunk < j->hi ? a + j->chunk : j->hi;
    tab_search_t s;
    memset(&s, 0, sizeof s);
    s.t = j->t;
    s.lo = a;
    s.hi = b;
    s.dump = j->dump ? j->dump + (a - j->lo) : NULL;
    tab_runs(&s, 0, 0);
    tab_merge(&loc, &s, j->t->n_windows);
  }
  pthread_mutex_lock(&j->mu);
  tab_merge(&j->acc, &loc, j->t->n_windows);
  pthread_mutex_unlock(&j->mu);
  return NULL;
}

/* constrained_search over ranks [lo, hi) for several windows at once (one scan):
 * out_cost/out_rank[i] = the reference's (cost, rank) winner for windows[i]
 * (out_rank = -1 when no layout is memory-feasible); *feasible = memory-feasible layouts;
 * dump (optional, hi-lo doubles): per_step of every rank (+inf when infeasible). */
int or_constrained_search_tab(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                              const int32_t* ids, int32_t n, const gp_train_opts* opts,
                              const int32_t* windows, int32_t n_windows, int64_t lo, int64_t hi,
                              int32_t threads, double* out_cost, int64_t* out_rank,
                              int64_t* feasible, int64_t* layouts, double* dump) {
  if (n <= 0) return fail(GP_INVALID, "constrained_search requires a non-empty train set");
  if (n_windows < 1 || n_windows > TAB_MAX_WINDOWS) return fail(GP_INVALID, "1..8 windows");
  layout_space_t sp;
  int rc = space_build(&sp, c, w, ids, n, opts);
  if (rc) return rc;
  int64_t total = count_layouts(&sp);
  if (hi < 0 || hi > total) hi = total;
  if (lo < 0) lo = 0;
  *layouts = total;
  tab_t t;
  tab_build(&t, &sp, w, k);
  t.n_windows = n_windows;
  t.windows = windows;
  tab_job_t job;
  memset(&job, 0, sizeof job);
  job.t = &t;
  job.lo = lo;
  job.hi = hi;
  job.dump = dump;
  if (threads < 1) threads = 1;
  int64_t span = hi > lo ? hi - lo : 0;
  job.chunk = span / (threads * 64) + 1;
  if (job.chunk < 4096) job.chunk = 4096;
  atomic_init(&job.next, lo);
  pthread_mutex_init(&job.mu, NULL);
  if (sp.max_stages >= sp.n_runs && lo < hi) {
    pthread_t th[256];
    if (threads > 256) threads = 256;
    for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, tab_worker, &job);
    for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  }
  pthread_mutex_destroy(&job.mu);
  *feasible = job.acc.feasible;
  for (int i = 0; i < n_windows; ++i) {
    out_cost[i] = job.acc.have[i] ? job.acc.best_cost[i] : 0.0;
    out_rank[i] = job.acc.have[i] ? job.acc.best_rank[i] : -1;
  }
  tab_free(&t);
  space_free(&sp);
  return GP_OK;
}

/* per_step of the layouts of several rank ranges [lo[i], hi[i]) (concatenated into out),
 * the memoised tables built once (as or_constrained_search_tab's dump). */
int or_layout_costs_tab(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                        const int32_t* ids, int32_t n, const gp_train_opts* opts, int32_t n_ranges,
                        const int64_t* lo, const int64_t* hi, double* out) {
  if (n <= 0) return fail(GP_INVALID, "constrained_search requires a non-empty train set");
  layout_space_t sp;
  int rc = space_build(&sp, c, w, ids, n, opts);
  if (rc) return rc;
  int64_t total = count_layouts(&sp);
  tab_t t;
  tab_build(&t, &sp, w, k);
  int32_t one = 1;
  t.n_windows = 1;
  t.windows = &one;
  size_t off = 0;
  for (int i = 0; i < n_ranges && !rc; ++i) {
    if (lo[i] < 0 || hi[i] > total || lo[i] > hi[i]) {
      rc = fail(GP_INVALID, "rank range outside the layout space");
      break;
    }
    tab_search_t s;
    memset(&s, 0, sizeof s);
    s.t = &t;
    s.lo = lo[i];
    s.hi = hi[i];
    s.dump = out + off;
    if (sp.max_stages >= sp.n_runs && lo[i] < hi[i]) tab_runs(&s, 0, 0);
    off += (size_t)(hi[i] - lo[i]);
  }
  tab_free(&t);
  space_free(&sp);
  return rc;
}
