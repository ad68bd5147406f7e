/* oracle_sched.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * rlsched repartition solver (src/partition.cpp) and the Algorithm-1 driver
 * (src/scheduler.cpp). Parity checker for the B200 engine; never shipped.
 */
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

#define K_INF 1e30

int or__fail(int code, const char* fmt, ...); /* oracle.c: shared last-error buffer */
#define fail2 or__fail

static double lnk(const gp_cluster* c, int a, int b) {
  return c->links[(size_t)a * (size_t)c->n_devices + (size_t)b];
}

/* ---------------------------------------------------------- SplitMix64 */
/* inc/common.hpp:71-90 */
typedef struct {
  uint64_t s;
} smx_t;
static uint64_t smx_next(smx_t* r) {
  uint64_t z = (r->s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static double smx_double(smx_t* r) { return (double)(smx_next(r) >> 11) * 0x1.0p-53; }

/* ---------------------------------------------------------- units */
/* build_units (src/partition.cpp:37-80) */
typedef struct {
  int n;
  int** members;
  int* n_members;
  double *flops, *hbm, *internal;
  double* cross;  /* n*n */
  double total_flops, total_hbm, total_link;
} units_t;

static void units_free(units_t* u) {
  for (int i = 0; i < u->n; ++i) free(u->members[i]);
  free(u->members);
  free(u->n_members);
  free(u->flops);
  free(u->hbm);
  free(u->internal);
  free(u->cross);
}

static void units_build(units_t* u, const gp_cluster* c, int machine_gran) {
  int by_machine = machine_gran && c->n_machines >= 2;
  int n = by_machine ? c->n_machines : c->n_devices;
  u->n = n;
  u->members = (int**)calloc((size_t)n, sizeof(int*));
  u->n_members = (int*)calloc((size_t)n, sizeof(int));
  for (int i = 0; i < n; ++i) u->members[i] = (int*)malloc(sizeof(int) * (size_t)c->n_devices);
  if (by_machine) {
    /* MachineInfo::device_ids: devices of machine m in creation (id) order */
    for (int d = 0; d < c->n_devices; ++d) {
      int m = c->device_machine[d];
      u->members[m][u->n_members[m]++] = d;
    }
  } else {
    for (int d = 0; d < n; ++d) {
      u->members[d][0] = d;
      u->n_members[d] = 1;
    }
  }
  u->flops = (double*)calloc((size_t)n, sizeof(double));
  u->hbm = (double*)calloc((size_t)n, sizeof(double));
  u->internal = (double*)calloc((size_t)n, sizeof(double));
  u->cross = (double*)calloc((size_t)n * (size_t)n, sizeof(double));
  for (int i = 0; i < n; ++i) {
    for (int a = 0; a < u->n_members[i]; ++a) {
      int da = u->members[i][a];
      u->flops[i] += c->device_flops[da];
      u->hbm[i] += c->device_hbm_bw[da];
      for (int b = a + 1; b < u->n_members[i]; ++b) u->internal[i] += lnk(c, da, u->members[i][b]);
    }
    for (int j = i + 1; j < n; ++j) {
      double bw = 0;
      for (int a = 0; a < u->n_members[i]; ++a)
        for (int b = 0; b < u->n_members[j]; ++b) bw += lnk(c, u->members[i][a], u->members[j][b]);
      u->cross[(size_t)i * n + j] = u->cross[(size_t)j * n + i] = bw;
    }
  }
  u->total_flops = 0.0;
  u->total_hbm = 0.0;
  for (int i = 0; i < n; ++i) u->total_flops += u->flops[i];
  for (int i = 0; i < n; ++i) u->total_hbm += u->hbm[i];
  u->total_link = 0;
  for (int i = 0; i < n; ++i) {
    u->total_link += u->internal[i];
    for (int j = i + 1; j < n; ++j) u->total_link += u->cross[(size_t)i * n + j];
  }
}

/* ---------------------------------------------------------- State */
/* State (src/partition.cpp:83-163) */
typedef struct {
  const units_t* u;
  char* in_train;
  double* ltt;
  double link_train, hbm_train, flops_train;
  int count;
} state_t;

static void st_init(state_t* s, const units_t* u) {
  s->u = u;
  s->in_train = (char*)calloc((size_t)u->n, 1);
  s->ltt = (double*)calloc((size_t)u->n, sizeof(double));
  s->link_train = s->hbm_train = s->flops_train = 0;
  s->count = 0;
}
static void st_free(state_t* s) {
  free(s->in_train);
  free(s->ltt);
}
static void st_add(state_t* s, int i) {
  const units_t* u = s->u;
  s->link_train += s->ltt[i] + u->internal[i];
  s->hbm_train += u->hbm[i];
  s->flops_train += u->flops[i];
  s->count++;
  s->in_train[i] = 1;
  for (int j = 0; j < u->n; ++j)
    if (j != i) s->ltt[j] += u->cross[(size_t)i * u->n + j];
}
static void st_remove(state_t* s, int i) {
  const units_t* u = s->u;
  s->in_train[i] = 0;
  for (int j = 0; j < u->n; ++j)
    if (j != i) s->ltt[j] -= u->cross[(size_t)i * u->n + j];
  s->link_train -= s->ltt[i] + u->internal[i];
  s->hbm_train -= u->hbm[i];
  s->flops_train -= u->flops[i];
  s->count--;
}
static double st_obj(const state_t* s) {
  const units_t* u = s->u;
  double lf = u->total_link > 0 ? s->link_train / u->total_link : 0;
  return lf + (u->total_hbm - s->hbm_train) / u->total_hbm;
}
static double st_frac(const state_t* s) { return s->flops_train / s->u->total_flops; }
static double st_obj_move(const state_t* s, int i, int to_train) {
  const units_t* u = s->u;
  double lt = s->link_train;
  if (to_train) lt += s->ltt[i] + u->internal[i];
  else lt -= s->ltt[i] + u->internal[i];
  double hbm = s->hbm_train + (to_train ? u->hbm[i] : -u->hbm[i]);
  double lf = u->total_link > 0 ? lt / u->total_link : 0;
  return lf + (u->total_hbm - hbm) / u->total_hbm;
}
static double st_frac_move(const state_t* s, int i, int to_train) {
  return (s->flops_train + (to_train ? s->u->flops[i] : -s->u->flops[i])) / s->u->total_flops;
}
static double st_obj_swap(const state_t* s, int a, int b) {
  const units_t* u = s->u;
  double lt = s->link_train - (s->ltt[a] + u->internal[a]) + (s->ltt[b] + u->internal[b]) -
              u->cross[(size_t)a * u->n + b];
  double hbm = s->hbm_train - u->hbm[a] + u->hbm[b];
  double lf = u->total_link > 0 ? lt / u->total_link : 0;
  return lf + (u->total_hbm - hbm) / u->total_hbm;
}
static double st_frac_swap(const state_t* s, int a, int b) {
  return (s->flops_train - s->u->flops[a] + s->u->flops[b]) / s->u->total_flops;
}
static int cmp_int(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}
/* train_devices (src/partition.cpp:155-162); returns count */
static int st_train_devices(const state_t* s, int* out) {
  int n = 0;
  for (int i = 0; i < s->u->n; ++i)
    if (s->in_train[i])
      for (int a = 0; a < s->u->n_members[i]; ++a) out[n++] = s->u->members[i][a];
  qsort(out, (size_t)n, sizeof(int), cmp_int);
  return n;
}

typedef struct {
  double lo, hi;
} band_t;
static int band_has(band_t b, double f) { return f >= b.lo && f <= b.hi; }

/* ---------------------------------------------------------- TopK */
/* TopK (src/partition.cpp:174-210) */
typedef struct {
  double obj;
  int* foot;   /* n_machines */
  int* train;
  int nt;
} tk_entry_t;
typedef struct {
  int k, n_machines, n_dev;
  const gp_cluster* c;
  tk_entry_t* items;
  int n;
} topk_t;

static int lex_less(const int* a, int na, const int* b, int nb) {
  int m = na < nb ? na : nb;
  for (int i = 0; i < m; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return na < nb;
}
static int tk_before(const tk_entry_t* a, const tk_entry_t* b) {
  if (a->obj != b->obj) return a->obj > b->obj;
  return lex_less(a->train, a->nt, b->train, b->nt);
}
static void tk_offer(topk_t* t, double obj, const int* train, int nt) {
  int* foot = (int*)calloc((size_t)t->n_machines, sizeof(int));
  for (int i = 0; i < nt; ++i) foot[t->c->device_machine[train[i]]]++;
  for (int e = 0; e < t->n; ++e) {
    tk_entry_t* it = &t->items[e];
    if (fabs(it->obj - obj) <= 1e-12 && memcmp(it->foot, foot, sizeof(int) * (size_t)t->n_machines) == 0) {
      if (lex_less(train, nt, it->train, it->nt)) {
        memcpy(it->train, train, sizeof(int) * (size_t)nt);
        it->nt = nt;
      }
      free(foot);
      return;
    }
  }
  tk_entry_t ne;
  ne.obj = obj;
  ne.foot = foot;
  ne.train = (int*)malloc(sizeof(int) * (size_t)(t->n_dev > 0 ? t->n_dev : 1));
  memcpy(ne.train, train, sizeof(int) * (size_t)nt);
  ne.nt = nt;
  /* push_back + std::sort of the whole list: a merge above does not re-sort, so
   * the list may be out of order until the next push (reference behaviour).
   * (objective desc, train asc) is a strict total order -> any sort agrees. */
  t->items[t->n++] = ne;
  for (int i = 1; i < t->n; ++i) {
    tk_entry_t cur = t->items[i];
    int j = i;
    while (j > 0 && tk_before(&cur, &t->items[j - 1])) {
      t->items[j] = t->items[j - 1];
      --j;
    }
    t->items[j] = cur;
  }
  if (t->n > t->k) {
    t->n--;
    free(t->items[t->n].foot);
    free(t->items[t->n].train);
  }
}

/* ---------------------------------------------------------- solvers */
/* exact_enumeration (src/partition.cpp:212-222) */
static void exact_enum(const units_t* u, band_t band, topk_t* tk, int* buf) {
  int n = u->n;
  for (uint64_t mask = 1; mask + 1 < (1ull << n); ++mask) {
    state_t s;
    st_init(&s, u);
    for (int i = 0; i < n; ++i)
      if (mask & (1ull << i)) st_add(&s, i);
    if (band_has(band, st_frac(&s))) {
      int nt = st_train_devices(&s, buf);
      tk_offer(tk, st_obj(&s), buf, nt);
    }
    st_free(&s);
  }
}

/* greedy_seed (src/partition.cpp:224-269) */
static int greedy_seed(state_t* st, band_t band, const int* order, double target) {
  const units_t* u = st->u;
  const int n = u->n;
  for (int oi = 0; oi < n; ++oi) {
    if (st_frac(st) >= target) break;
    if (st->count + 1 >= n) break;
    st_add(st, order[oi]);
  }
  for (int guard = 0; guard < 4 * n; ++guard) {
    double f = st_frac(st);
    if (band_has(band, f)) break;
    if (f > band.hi) {
      if (st->count <= 1) return 0;
      int pick = n;
      for (int i = 0; i < n; ++i)
        if (st->in_train[i] && (pick == n || u->flops[i] < u->flops[pick])) pick = i;
      st_remove(st, pick);
    } else {
      if (st->count + 1 >= n) return 0;
      int pick = n;
      for (int oi = 0; oi < n; ++oi) {
        int i = order[oi];
        if (st->in_train[i]) continue;
        if (st_frac_move(st, i, 1) <= band.hi + 1e-15) {
          pick = i;
          break;
        }
      }
      if (pick == n) {
        for (int i = 0; i < n; ++i)
          if (!st->in_train[i] && (pick == n || u->flops[i] < u->flops[pick])) pick = i;
        if (pick == n) return 0;
      }
      st_add(st, pick);
    }
  }
  return band_has(band, st_frac(st)) && st->count > 0 && st->count < n;
}

typedef struct {
  int idx;
  double score;
} ord_t;
static double* g_scores;
static int cmp_score_desc_stable(const void* pa, const void* pb) {
  int a = *(const int*)pa, b = *(const int*)pb;
  if (g_scores[a] > g_scores[b]) return -1;
  if (g_scores[a] < g_scores[b]) return 1;
  return (a > b) - (a < b); /* stable: original (index) order */
}

/* local_search (src/partition.cpp:271-350) */
/* move/swap candidates examined by local_search (the U3 work unit): per ascent
 * step n moves + |train| * |rollout| swaps; test infrastructure, not thread-safe */
static int64_t g_part_evals;
int64_t or_partition_evals(int reset) {
  const int64_t v = g_part_evals;
  if (reset) g_part_evals = 0;
  return v;
}

static void local_search(const units_t* u, band_t band, const gp_part_opts* o, topk_t* tk, int* buf) {
  int n = u->n;
  double* base = (double*)malloc(sizeof(double) * (size_t)n);
  double* score = (double*)malloc(sizeof(double) * (size_t)n);
  int* order = (int*)malloc(sizeof(int) * (size_t)n);
  for (int i = 0; i < n; ++i) {
    double d = 0;
    for (int j = 0; j < n; ++j)
      if (j != i) d += u->cross[(size_t)i * n + j];
    d += 2.0 * u->internal[i];
    if (n > 1) d /= (double)(n - 1);
    base[i] = d * u->flops[i];
  }
  for (int r = 0; r < o->restarts; ++r) {
    smx_t rng = {o->seed + (uint64_t)r * 0x9e3779b97f4a7c15ull};
    for (int i = 0; i < n; ++i) {
      order[i] = i;
      score[i] = base[i];
    }
    if (r > 0)
      for (int i = 0; i < n; ++i) score[i] *= 0.5 + smx_double(&rng);
    g_scores = score;
    qsort(order, (size_t)n, sizeof(int), cmp_score_desc_stable);
    double bhi = (1.0 < band.hi) ? 1.0 : band.hi; /* std::min(band.hi, 1.0) */
    double blo = (band.lo < 0.0) ? 0.0 : band.lo; /* std::max(band.lo, 0.0) */
    double target = blo + (r + 0.5) / o->restarts * (bhi - blo);
    state_t st;
    st_init(&st, u);
    if (!greedy_seed(&st, band, order, target)) {
      st_free(&st);
      continue;
    }
    for (;;) {
      double cur = st_obj(&st);
      double best_gain = 1e-12;
      g_part_evals += n + (int64_t)st.count * (n - st.count);
      int kind = -1, mi = 0, mj = 0;
      for (int i = 0; i < n; ++i) {
        int to_train = !st.in_train[i];
        if (to_train && st.count + 1 == n) continue;
        if (!to_train && st.count == 1) continue;
        if (!band_has(band, st_frac_move(&st, i, to_train))) continue;
        double gain = st_obj_move(&st, i, to_train) - cur;
        if (gain > best_gain) {
          best_gain = gain;
          kind = 0;
          mi = i;
        }
      }
      for (int a = 0; a < n; ++a) {
        if (!st.in_train[a]) continue;
        for (int b = 0; b < n; ++b) {
          if (st.in_train[b]) continue;
          if (!band_has(band, st_frac_swap(&st, a, b))) continue;
          double gain = st_obj_swap(&st, a, b) - cur;
          if (gain > best_gain) {
            best_gain = gain;
            kind = 1;
            mi = a;
            mj = b;
          }
        }
      }
      if (kind < 0) break;
      if (kind == 0) {
        if (st.in_train[mi]) st_remove(&st, mi);
        else st_add(&st, mi);
      } else {
        st_remove(&st, mi);
        st_add(&st, mj);
      }
    }
    int nt = st_train_devices(&st, buf);
    tk_offer(tk, st_obj(&st), buf, nt);
    st_free(&st);
  }
  free(base);
  free(score);
  free(order);
}

/* compute_fraction (src/partition.cpp:361-367) */
static double compute_fraction(const gp_cluster* c, const int* train, int nt) {
  double total = 0, tr = 0;
  for (int d = 0; d < c->n_devices; ++d) total += c->device_flops[d];
  for (int i = 0; i < nt; ++i) tr += c->device_flops[train[i]];
  return tr / total;
}

/* graph_partition_candidates (src/partition.cpp:369-406) */
int or_partition_candidates(const gp_cluster* c, const gp_gamma* g, const gp_part_opts* o, int32_t k,
                            gp_partition* out, int32_t* train_ids, int32_t* n_out) {
  *n_out = 0;
  if (c->n_devices < 2) return fail2(GP_INVALID, "graph_partition requires at least two devices");
  units_t u;
  units_build(&u, c, o->machine_granularity);
  band_t band = {g->gamma_l - o->band_epsilon, g->gamma_h + o->band_epsilon};
  topk_t tk = {k, c->n_machines, c->n_devices, c, NULL, 0};
  tk.items = (tk_entry_t*)calloc((size_t)k + 1, sizeof(tk_entry_t));
  int* buf = (int*)malloc(sizeof(int) * (size_t)c->n_devices);
  if (!o->force_local_search && u.n <= o->exact_threshold && u.n <= 20) exact_enum(&u, band, &tk, buf);
  else local_search(&u, band, o, &tk, buf);
  int rc = GP_OK;
  if (tk.n == 0) {
    rc = fail2(GP_BAND_INFEASIBLE, "no bisection satisfies the compute-fraction band [%f, %f]",
               g->gamma_l, g->gamma_h);
  } else {
    int off = 0;
    for (int e = 0; e < tk.n; ++e) {
      out[e].train_offset = off;
      out[e].train_count = tk.items[e].nt;
      out[e].objective = tk.items[e].obj;
      out[e].compute_fraction = compute_fraction(c, tk.items[e].train, tk.items[e].nt);
      memcpy(train_ids + off, tk.items[e].train, sizeof(int) * (size_t)tk.items[e].nt);
      off += tk.items[e].nt;
    }
    *n_out = tk.n;
  }
  for (int e = 0; e < tk.n; ++e) {
    free(tk.items[e].foot);
    free(tk.items[e].train);
  }
  free(tk.items);
  free(buf);
  units_free(&u);
  return rc;
}

/* partition_objective (src/partition.cpp:354-358) */
int or_partition_objective(const gp_cluster* c, const int32_t* train, int32_t nt, double* objective,
                           double* fraction) {
  units_t u;
  units_build(&u, c, 0);
  state_t s;
  st_init(&s, &u);
  for (int i = 0; i < nt; ++i) st_add(&s, train[i]);
  *objective = st_obj(&s);
  *fraction = compute_fraction(c, train, nt);
  st_free(&s);
  units_free(&u);
  return GP_OK;
}

/* ================================================================ driver */

typedef struct {
  int* train;
  int nt;
  int* roll;
  int nr;
  /* train side */
  int train_found;
  gp_train_result tr;
  int* stage_dev;  /* nt */
  /* rollout side */
  int roll_found;
  gp_rollout_result rr;
  gp_config* cfg;        /* entry configs, rr.n_entries */
  gp_rollout_entry* ent;
  /* CostEstimate */
  double c_train, c_rollout, c_reward, c_update, c_infer;
  int window;
} iter_t;

static int it_feasible(const iter_t* it) { return it->train_found && it->roll_found; }
static double it_objective(const iter_t* it) {
  return it->c_train < it->c_infer ? it->c_infer : it->c_train;
}

typedef struct {
  const gp_cluster* c;
  const gp_workload* w;
  const gp_calib* k;
  int window;
  iter_t** memo;
  int n_memo, cap_memo;
  int err;
  int tab_threads;  /* > 0: table-memoised constrained_search for spaces > 1e5 layouts */
} search_phase_t;

static int same_set(const int* a, int na, const int* b, int nb) {
  return na == nb && memcmp(a, b, sizeof(int) * (size_t)na) == 0;
}

/* evaluate_partition (src/scheduler.cpp:42-75) */
static int evaluate_partition(search_phase_t* sp, const int* train, int nt, const int* roll, int nr,
                              iter_t* it) {
  const gp_cluster* c = sp->c;
  const gp_workload* w = sp->w;
  memset(it, 0, sizeof *it);
  it->train = (int*)malloc(sizeof(int) * (size_t)nt);
  memcpy(it->train, train, sizeof(int) * (size_t)nt);
  it->nt = nt;
  it->roll = (int*)malloc(sizeof(int) * (size_t)nr);
  memcpy(it->roll, roll, sizeof(int) * (size_t)nr);
  it->nr = nr;
  it->window = sp->window;
  it->c_reward = w->reward_cost_const;
  gp_train_opts to = {4, 16};
  it->stage_dev = (int*)malloc(sizeof(int) * (size_t)(nt > 0 ? nt : 1));
  int rc;
  int64_t space = 0;
  if (sp->tab_threads > 0 && or_train_space(c, w, train, nt, &to, &space) == GP_OK && space > 100000) {
    /* table-memoised scan for the winner's rank, then the plain restatement on that one rank
     * for the plan (its cost is the same value) */
    double cost;
    int64_t rank, feasible, layouts;
    int32_t win = sp->window;
    rc = or_constrained_search_tab(c, w, sp->k, train, nt, &to, &win, 1, 0, -1, sp->tab_threads, &cost,
                                   &rank, &feasible, &layouts, NULL);
    if (rc) return rc;
    if (rank >= 0) {
      rc = or_constrained_search(c, w, sp->k, train, nt, sp->window, &to, rank, rank + 1, &it->tr,
                                 it->stage_dev);
      if (rc) return rc;
      it->tr.rank = rank;
      it->tr.cost = cost;
    } else {
      memset(&it->tr, 0, sizeof it->tr);
    }
    it->tr.layouts = layouts;
    it->tr.feasible = feasible;
  } else {
    rc = or_constrained_search(c, w, sp->k, train, nt, sp->window, &to, 0, -1, &it->tr, it->stage_dev);
  }
  if (rc) return rc;
  it->train_found = it->tr.found;
  double B = (double)w->batch_rollouts * sp->window;
  gp_rollout_opts ro = {4};
  int cap = 4096;
  gp_config* cfgs = (gp_config*)malloc(sizeof(gp_config) * (size_t)cap);
  int ncfg = 0;
  rc = or_enumerate_configs(c, w, sp->k, roll, nr, &ro, cfgs, cap, &ncfg);
  if (rc) {
    free(cfgs);
    return rc;
  }
  if (ncfg > 0) {
    int caps[GP_MAX_TYPES];
    or_rollout_capacities(c, roll, nr, caps);
    gp_rollout_entry* ent = (gp_rollout_entry*)malloc(sizeof(gp_rollout_entry) * (size_t)ncfg);
    rc = or_solve_milp(cfgs, ncfg, caps, c->n_types, B, w->mean_len, &it->rr, ent);
    if (rc == GP_OK) {
      it->roll_found = 1;
      it->cfg = (gp_config*)malloc(sizeof(gp_config) * (size_t)(it->rr.n_entries + 1));
      it->ent = ent;
      for (int e = 0; e < it->rr.n_entries; ++e) it->cfg[e] = cfgs[ent[e].config];
    } else {
      free(ent);
      if (rc != GP_INFEASIBLE) {
        free(cfgs);
        return rc;
      }
    }
  }
  free(cfgs);
  it->c_train = it->train_found ? it->tr.cost : K_INF;
  if (it->roll_found && it->train_found) {
    it->c_rollout = it->rr.makespan;
    int ne = it->rr.n_entries;
    int* et = (int*)malloc(sizeof(int) * (size_t)(ne + 1));
    int* er = (int*)malloc(sizeof(int) * (size_t)(ne + 1));
    for (int e = 0; e < ne; ++e) {
      et[e] = -1;
      for (int t = 0; t < c->n_types; ++t)
        if (it->cfg[e].type_counts[t] > 0) {
          et[e] = t;
          break;
        }
      er[e] = it->ent[e].replicas;
    }
    or_weight_sync_cost(c, w, sp->k, it->train, nt, it->roll, nr, et, er, ne, sp->window, &it->c_update);
    free(et);
    free(er);
    it->c_infer = it->c_rollout + it->c_reward + it->c_update;
  } else {
    it->c_rollout = it->roll_found ? it->rr.makespan : K_INF;
    it->c_infer = K_INF;
  }
  return GP_OK;
}

static void it_free(iter_t* it) {
  free(it->train);
  free(it->roll);
  free(it->stage_dev);
  free(it->cfg);
  free(it->ent);
}

/* SearchPhase::eval (src/scheduler.cpp:106-120): memo by train set. */
static iter_t* sp_eval(search_phase_t* sp, const int* train, int nt, const int* roll, int nr) {
  for (int i = 0; i < sp->n_memo; ++i)
    if (same_set(sp->memo[i]->train, sp->memo[i]->nt, train, nt)) return sp->memo[i];
  iter_t* it = (iter_t*)calloc(1, sizeof(iter_t));
  int rc = evaluate_partition(sp, train, nt, roll, nr, it);
  if (rc) {
    sp->err = rc;
    it_free(it);
    free(it);
    return NULL;
  }
  if (sp->n_memo == sp->cap_memo) {
    sp->cap_memo = sp->cap_memo ? 2 * sp->cap_memo : 64;
    sp->memo = (iter_t**)realloc(sp->memo, sizeof(iter_t*) * (size_t)sp->cap_memo);
  }
  sp->memo[sp->n_memo++] = it;
  return it;
}

/* BestTracker (src/scheduler.cpp:77-95); entries point into the memo. */
typedef struct {
  const iter_t* conforming;
  const iter_t* any;
} best_t;
static void best_offer(best_t* b, const iter_t* it) {
  if (!it || !it_feasible(it)) return;
  double m = it_objective(it);
  if (!b->any || m < it_objective(b->any)) b->any = it;
  if (it->c_infer >= it->c_train)
    if (!b->conforming || m < it_objective(b->conforming)) b->conforming = it;
}

typedef struct {
  double gl, gh;
  double q, r;
} gamma_t;

/* partition_with_widening (src/scheduler.cpp:21-40) -> candidate train sets. */
static int partition_with_widening(const gp_cluster* c, gamma_t g, const or_sched_opts* o,
                                   gp_partition* parts, int* ids, int* n_parts) {
  double widen = 0;
  gp_part_opts po = {12, o->restarts, o->seed, 1e-9, 0, 0};
  for (;;) {
    gp_gamma gg;
    gg.q = g.q;
    gg.r = g.r;
    double lo = g.gl - widen, hi = g.gh + widen;
    gg.gamma_l = (0.0 < lo) ? lo : 0.0; /* std::max(0.0, gl - widen) */
    gg.gamma_h = (hi < 1.0) ? hi : 1.0; /* std::min(1.0, gh + widen) */
    int rc = or_partition_candidates(c, &gg, &po, 8, parts, ids, n_parts);
    if (rc == GP_OK) return GP_OK;
    if (rc != GP_BAND_INFEASIBLE) return rc;
    if (gg.gamma_l <= 0.0 && gg.gamma_h >= 1.0)
      return fail2(GP_INFEASIBLE, "no feasible bisection exists even with an unconstrained band");
    widen += o->band_widen_step;
  }
}

static int complement(const gp_cluster* c, const int* train, int nt, int* roll) {
  char* in = (char*)calloc((size_t)c->n_devices, 1);
  for (int i = 0; i < nt; ++i) in[train[i]] = 1;
  int nr = 0;
  for (int d = 0; d < c->n_devices; ++d)
    if (!in[d]) roll[nr++] = d;
  free(in);
  return nr;
}

typedef struct {
  const iter_t* best;
  int iterations;
  int converged;
  double* trace;  /* 4 per iteration */
  int n_trace;
} run_t;

static int g_lead;
static const gp_cluster* g_lead_c;
static int cmp_lead(const void* pa, const void* pb) {
  int a = *(const int*)pa, b = *(const int*)pb;
  int ta = g_lead_c->device_type[a], tb = g_lead_c->device_type[b];
  int la = ta == g_lead, lb = tb == g_lead;
  if (la != lb) return la ? -1 : 1;
  if (ta != tb) return ta < tb ? -1 : 1;
  return (a > b) - (a < b);
}

/* run_two_phase (src/scheduler.cpp:122-255) */
static int run_two_phase(search_phase_t* sp, const or_sched_opts* o, run_t* run) {
  const gp_cluster* c = sp->c;
  const int N = c->n_devices;
  gamma_t gamma = {1, 1, 0, 1};
  int frozen = 0;
  best_t best = {NULL, NULL};
  const iter_t* cached = NULL;
  int reuse = 0;
  double anchor = 0;
  int has_anchor = 0, streak = 0;
  gp_partition parts[8];
  int* ids = (int*)malloc(sizeof(int) * (size_t)N * 8);
  int* roll = (int*)malloc(sizeof(int) * (size_t)N);
  int* order = (int*)malloc(sizeof(int) * (size_t)N);
  int* tset = (int*)malloc(sizeof(int) * (size_t)N);
  int rc = GP_OK;
  run->trace = (double*)malloc(sizeof(double) * 4 * 200);
  run->n_trace = 0;
  run->converged = 0;
  for (int iter = 1; iter <= 200; ++iter) {
    run->iterations = iter;
    const iter_t* it;
    if (reuse && cached) {
      it = cached;
    } else {
      int np = 0;
      rc = partition_with_widening(c, gamma, o, parts, ids, &np);
      if (rc) goto done;
      int nr = complement(c, ids + parts[0].train_offset, parts[0].train_count, roll);
      it = sp_eval(sp, ids + parts[0].train_offset, parts[0].train_count, roll, nr);
      if (!it) { rc = sp->err; goto done; }
      for (int p = 1; p < np; ++p) {
        nr = complement(c, ids + parts[p].train_offset, parts[p].train_count, roll);
        const iter_t* e = sp_eval(sp, ids + parts[p].train_offset, parts[p].train_count, roll, nr);
        if (!e) { rc = sp->err; goto done; }
        best_offer(&best, e);
      }
      if (iter == 1) {
        for (int p = 1; p <= 15; ++p) {
          gamma_t probe = gamma;
          probe.gl = probe.gh = (double)p / (15 + 1);
          gp_partition pp[8];
          int npp = 0;
          int* pids = (int*)malloc(sizeof(int) * (size_t)N * 8);
          rc = partition_with_widening(c, probe, o, pp, pids, &npp);
          if (rc) { free(pids); goto done; }
          for (int q = 0; q < npp; ++q) {
            nr = complement(c, pids + pp[q].train_offset, pp[q].train_count, roll);
            const iter_t* e = sp_eval(sp, pids + pp[q].train_offset, pp[q].train_count, roll, nr);
            if (!e) { rc = sp->err; free(pids); goto done; }
            best_offer(&best, e);
          }
          free(pids);
        }
        for (int lead = 0; lead < c->n_types; ++lead) {
          for (int d = 0; d < N; ++d) order[d] = d;
          g_lead = lead;
          g_lead_c = c;
          qsort(order, (size_t)N, sizeof(int), cmp_lead);
          for (int m = 0; m + 1 < N; ++m) {
            for (int i = 0; i <= m; ++i) tset[i] = order[i];
            qsort(tset, (size_t)(m + 1), sizeof(int), cmp_int);
            nr = 0;
            for (int i = m + 1; i < N; ++i) roll[nr++] = order[i];
            qsort(roll, (size_t)nr, sizeof(int), cmp_int);
            const iter_t* e = sp_eval(sp, tset, m + 1, roll, nr);
            if (!e) { rc = sp->err; goto done; }
            best_offer(&best, e);
          }
        }
      }
      cached = it;
    }
    best_offer(&best, it);
    double m = it_objective(it);
    double* tr = run->trace + 4 * run->n_trace++;
    tr[0] = (gamma.gl + gamma.gh) / 2;
    tr[1] = it->c_train;
    tr[2] = it->c_infer;
    tr[3] = m;
    if (has_anchor && fabs(m - anchor) <= 0.005 * fabs(anchor)) {
      streak++;
    } else {
      anchor = m;
      has_anchor = 1;
      streak = 0;
    }
    if (streak >= 20) {
      run->converged = 1;
      break;
    }
    if (!frozen) {
      double ct = it->c_train, ci = it->c_infer;
      double mx = ct < ci ? ci : ct;
      int balanced = it_feasible(it) && fabs(ct - ci) <= 0.02 * mx;
      if (balanced || (gamma.r - gamma.q) < 1e-3) {
        frozen = 1;
      } else if (iter == 1) {
        gamma.gl = gamma.gh = (gamma.q + gamma.r) / 2;
        cached = NULL;
      } else {
        /* refine_gamma (src/partition.cpp:10-20) */
        if (ct < ci) gamma.r = (gamma.q + gamma.r) / 2.0;
        else gamma.q = (gamma.q + gamma.r) / 2.0;
        double mid = (gamma.q + gamma.r) / 2.0;
        gamma.gl = gamma.gh = mid;
        cached = NULL;
      }
    }
    reuse = frozen && cached;
  }
  run->best = best.conforming ? best.conforming : best.any;
  if (!run->best)
    rc = fail2(GP_INFEASIBLE, "no feasible plan at any visited partition");
done:
  free(ids);
  free(roll);
  free(order);
  free(tset);
  return rc;
}

/* -------------------------------------------------------------- JSON out */
typedef struct {
  char* buf;
  size_t n, cap;
} sbuf_t;
static void sb_put(sbuf_t* s, const char* fmt, ...) {
  va_list ap;
  for (;;) {
    va_start(ap, fmt);
    int need = vsnprintf(s->buf + s->n, s->cap - s->n, fmt, ap);
    va_end(ap);
    if ((size_t)need < s->cap - s->n) {
      s->n += (size_t)need;
      return;
    }
    s->cap = 2 * s->cap + (size_t)need + 64;
    s->buf = (char*)realloc(s->buf, s->cap);
  }
}
static void sb_ints(sbuf_t* s, const int* v, int n) {
  sb_put(s, "[");
  for (int i = 0; i < n; ++i) sb_put(s, i ? ",%d" : "%d", v[i]);
  sb_put(s, "]");
}

static void free_memo(search_phase_t* sp) {
  for (int i = 0; i < sp->n_memo; ++i) {
    it_free(sp->memo[i]);
    free(sp->memo[i]);
  }
  free(sp->memo);
  sp->memo = NULL;
  sp->n_memo = sp->cap_memo = 0;
}

/* schedule (src/scheduler.cpp:259-292) */
int or_schedule(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                const or_sched_opts* o, char** plan_json) {
  *plan_json = NULL;
  if (c->n_devices < 2) return fail2(GP_INFEASIBLE, "scheduling requires at least two devices");
  int eta = o->eta_override >= 0 ? o->eta_override : w->staleness;
  gp_workload eff = *w;
  eff.staleness = eta;
  /* WindowExpander (inc/rollout_milp.hpp:51-81), cap 64, tol 0.01 */
  const int cap = 64;
  int delta = eta + 1;
  if (delta < 1) delta = 1;
  if (delta > cap) delta = cap;
  double last = 0;
  int has_last = 0, wstreak = 0;
  search_phase_t sp;
  run_t run;
  memset(&run, 0, sizeof run);
  for (;;) {
    memset(&sp, 0, sizeof sp);
    sp.c = c;
    sp.w = &eff;
    sp.k = k;
    sp.window = delta;
    sp.tab_threads = o->tab_threads;
    free(run.trace);
    memset(&run, 0, sizeof run);
    int rc = run_two_phase(&sp, o, &run);
    if (rc) {
      free(run.trace);
      free_memo(&sp);
      return rc;
    }
    double per_step = it_objective(run.best) / delta;
    int stop;
    {
      int stable = has_last && fabs(per_step - last) <= 0.01 * fabs(last);
      wstreak = stable ? wstreak + 1 : 0;
      last = per_step;
      has_last = 1;
      stop = wstreak >= 2 || delta >= cap;
    }
    if (!o->expand_window || stop) break;
    free_memo(&sp);
    delta = 2 * delta < cap ? 2 * delta : cap;
  }
  const iter_t* b = run.best;
  sbuf_t s = {(char*)malloc(4096), 0, 4096};
  sb_put(&s, "{\"window_steps\":%d,\"staleness\":%d,\"iterations_run\":%d,\"converged\":%s,", delta,
         eta, run.iterations, run.converged ? "true" : "false");
  sb_put(&s, "\"partition\":{\"train\":");
  sb_ints(&s, b->train, b->nt);
  sb_put(&s, ",\"rollout\":");
  sb_ints(&s, b->roll, b->nr);
  sb_put(&s, "},\"train_plan\":{\"stages\":[");
  for (int st = 0; st < b->tr.n_stages; ++st) {
    sb_put(&s, st ? ",{\"devices\":" : "{\"devices\":");
    sb_ints(&s, b->stage_dev + b->tr.stage[st].first, b->tr.stage[st].count);
    sb_put(&s, ",\"tp\":%d,\"dp\":%d,\"layers\":%d}", b->tr.stage[st].tp, b->tr.stage[st].dp,
           b->tr.stage[st].layers);
  }
  sb_put(&s, "],\"cost_s\":%.17g},\"rollout_plan\":{\"entries\":[", b->tr.cost);
  for (int e = 0; e < b->rr.n_entries; ++e) {
    const gp_config* cf = &b->cfg[e];
    sb_put(&s, e ? ",{\"type_counts\":" : "{\"type_counts\":");
    sb_ints(&s, cf->type_counts, c->n_types);
    sb_put(&s, ",\"tp_per_stage\":");
    sb_ints(&s, cf->tp, cf->n_stages);
    sb_put(&s, ",\"throughput_tps\":%.17g,\"machine_footprint\":", cf->throughput);
    sb_ints(&s, cf->tp, cf->n_stages);
    sb_put(&s, ",\"replicas\":%d,\"workload_rollouts\":%.17g}", b->ent[e].replicas, b->ent[e].workload);
  }
  sb_put(&s, "],\"makespan_s\":%.17g,\"total_rollouts\":%.17g},", b->rr.makespan, b->rr.total_rollouts);
  sb_put(&s,
         "\"costs\":{\"train_s\":%.17g,\"rollout_s\":%.17g,\"reward_s\":%.17g,\"update_s\":%.17g,"
         "\"infer_total_s\":%.17g,\"window_steps\":%d},",
         b->c_train, b->c_rollout, b->c_reward, b->c_update, b->c_infer, b->window);
  sb_put(&s, "\"trace\":[");
  for (int i = 0; i < run.n_trace; ++i)
    sb_put(&s, i ? ",[%.17g,%.17g,%.17g,%.17g]" : "[%.17g,%.17g,%.17g,%.17g]", run.trace[4 * i],
           run.trace[4 * i + 1], run.trace[4 * i + 2], run.trace[4 * i + 3]);
  sb_put(&s, "],\"evaluated_partitions\":%d}", sp.n_memo);
  *plan_json = s.buf;
  free(run.trace);
  free_memo(&sp);
  return GP_OK;
}
