// rollout.cu — sm_100a kernels for the rollout side of the hot path:
//   K3  enumerate_configs + replica_concurrency/replica_rate_at
//       (src/rollout_milp.cpp:39-89, src/cost_model.cpp:128-172)
//   K4  solve_milp: exact unbounded-knapsack DP over the type-capacity lattice
//       (src/rollout_milp.cpp:91-171), level-synchronous wavefront
//   K6  weight_sync_cost (src/cost_model.cpp:174-196)
//
// K4 design. best[s] = max_c best[s - v_c] + h_c with strict '>' in config order
// (first maximal config wins). Every config is type-pure and uses >= 1 device,
// so a state at level l = sum_t s_t depends only on lower levels: one level is
// one parallel step. Configs sharing (type, devices) read the same predecessor,
// and fp addition is monotone, so the value is max over groups of
// best[prev_g] + hmax_g (exact); the choice is the smallest config index c with
// best[prev_g(c)] + h_c == that value, found by scanning only the groups that
// reach it. The value and the choice are therefore identical to the reference's
// sequential scan; the backtracking walk runs on one device thread.
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "gp_internal.h"

namespace cg = cooperative_groups;

namespace gp {

// ------------------------------------------------------------------ K3 configs
constexpr int kAv = GP_MAX_ROLLOUT_STAGES;  // largest per-machine counts kept per type (one per stage)

struct CfgCand {
  int type;
  int stages;
  int tp[kAv];
  int set;  // rollout set of this candidate (batched enumeration)
};

__device__ __forceinline__ int trunc_i32_x86(double x) {
  // static_cast<int>(double) on x86-64 (cvttsd2si): out of range / NaN -> INT_MIN
  if (!(x > -2147483649.0 && x < 2147483648.0)) return INT_MIN;
  return static_cast<int>(x);
}

// One thread per (type, tp-multiset) candidate; the caller compacts in order.
__global__ void k3_configs(const CfgCand* __restrict__ cands, int n_cands,
                           const int* __restrict__ avail /* [T][kAv] largest machine counts */,
                           const int* __restrict__ n_machines /* [T] */, int max_stages,
                           Scalars sc, const double* __restrict__ tcap,
                           const double* __restrict__ thbm, const double* __restrict__ tflops,
                           const double* __restrict__ ceff, const double* __restrict__ ioeff,
                           int T, gp_config* __restrict__ out, int* __restrict__ keep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_cands) return;
  const CfgCand c = cands[i];
  const int t = c.type, S = c.stages;
  const int* nm = n_machines + c.set * T;
  const int* av = avail + c.set * T * kAv;
  int ms = max_stages < nm[t] ? max_stages : nm[t];
  ms = ms < sc.L ? ms : sc.L;
  bool ok = nm[t] > 0 && S <= ms;
  for (int s = 0; s < S && ok; ++s) ok = c.tp[s] <= av[t * kAv + s];  // stage k on k-th largest machine
  int conc = 0;
  if (ok) {
    // replica_concurrency (src/cost_model.cpp:128-148)
    int best = sc.max_conc;
    for (int s = 0; s < S; ++s) {
      const int layers = sc.L / S + (s < sc.L % S ? 1 : 0);  // layers_for_stage
      const int tp = c.tp[s];
      const double lf = static_cast<double>(layers) / sc.L;
      const double weight = sc.P * lf * sc.bpp_infer / tp;
      const double free_b = tcap[t] - weight;
      if (free_b < 0) {
        best = 0;
        break;
      }
      const double kv = sc.kvbpt * sc.mtl * lf / tp;
      if (kv > 0) {
        const int v = trunc_i32_x86(free_b / kv);
        best = v < best ? v : best;
      }
    }
    conc = best > 0 ? best : 0;
  }
  keep[i] = ok && conc >= 1;
  if (!keep[i]) return;
  gp_config cfg;
  for (int u = 0; u < GP_MAX_TYPES; ++u) cfg.type_counts[u] = 0;
  for (int u = 0; u < GP_MAX_ROLLOUT_STAGES; ++u) cfg.tp[u] = 0;
  int n = 0;
  for (int s = 0; s < S; ++s) {
    cfg.tp[s] = c.tp[s];
    n += c.tp[s];
  }
  cfg.type_counts[t] = n;
  cfg.n_stages = S;
  // replica_rate_at (src/cost_model.cpp:150-165): only type t contributes
  double agg_bw = 0, agg_flops = 0;
  for (int u = 0; u < T; ++u) {
    if (cfg.type_counts[u] == 0) continue;
    agg_bw += cfg.type_counts[u] * thbm[u] * ioeff[u];
    agg_flops += cfg.type_counts[u] * tflops[u] * ceff[u];
  }
  const double io_rate = static_cast<double>(conc) * agg_bw / sc.mbi;
  const double compute_rate = agg_flops / sc.ifpt;
  const double penalty = 1.0 + sc.stage_pen * (S - 1);
  const double m = compute_rate < io_rate ? compute_rate : io_rate;
  cfg.throughput = m / penalty;
  out[i] = cfg;
}

// ---------------------------------------------------------------- K4 MILP DP
struct MilpDims {
  int T;
  long long states;
  long long stride[GP_MAX_TYPES];
  int cap[GP_MAX_TYPES];
  int off[GP_MAX_TYPES];        // bit offset of coordinate t in the packed state word
  unsigned mask[GP_MAX_TYPES];  // (1 << bits_t) - 1
  int levels;                   // sum cap + 1
};

struct Group {
  int type;
  int n;             // devices of the type used by each member
  long long delta;   // n * stride[type]: predecessor offset
  double hmax;       // max member throughput
  int first, count;  // members[first .. first+count) = config indices, ascending
};

constexpr int kMaxGroups = 256;
constexpr int kMaxCfg = 1024;

__device__ __forceinline__ unsigned long long pack_state(const MilpDims& d, long long s, int& level) {
  unsigned long long pk = 0;
  level = 0;
  for (int t = d.T - 1; t >= 0; --t) {
    const int c = (int)(s / d.stride[t]);
    s -= (long long)c * d.stride[t];
    level += c;
    pk |= (unsigned long long)c << d.off[t];
  }
  return pk;
}

__global__ void k4_level_hist(MilpDims d, int* __restrict__ hist) {
  for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < d.states;
       s += (long long)gridDim.x * blockDim.x) {
    int l;
    pack_state(d, s, l);
    atomicAdd(&hist[l], 1);
  }
}

// exclusive scan of level counts (levels <= N+1, one thread)
__global__ void k4_level_scan(const int* __restrict__ hist, int levels, long long* __restrict__ off,
                              int* __restrict__ cursor, int* __restrict__ max_width) {
  if (threadIdx.x == 0) {
    long long acc = 0;
    int mw = 0;
    for (int l = 0; l < levels; ++l) {
      off[l] = acc;
      cursor[l] = 0;
      acc += hist[l];
      mw = hist[l] > mw ? hist[l] : mw;
    }
    off[levels] = acc;
    *max_width = mw;
  }
}

// states of each level, as packed coordinates (order within a level is irrelevant:
// a level's states read only lower levels)
__global__ void k4_level_scatter(MilpDims d, const long long* __restrict__ off,
                                 int* __restrict__ cursor, unsigned long long* __restrict__ order) {
  for (long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x; s < d.states;
       s += (long long)gridDim.x * blockDim.x) {
    int l;
    const unsigned long long pk = pack_state(d, s, l);
    const int slot = atomicAdd(&cursor[l], 1);
    order[off[l] + slot] = pk;
  }
}

// Lattice DP (k4_dp_multi below): one warp per state, lanes over the (type, devices)
// groups: value = max_g best[s - delta_g] + hmax_g; choice = smallest config index c with
// best[prev_g(c)] + h_c == value (src/rollout_milp.cpp:115-143). The lanes' partial
// (max value, min index) pairs merge exactly in any order. A state at level l reads levels
// <= l - n_min (n_min = fewest devices of any config), so `step` = n_min consecutive levels
// form one phase between grid barriers.
// Several lattice tables in one cooperative launch: phase p runs levels
// [p*step_t, (p+1)*step_t) of every table t (tables are independent), so a scheduler batch
// pays max_t(phases_t) grid barriers instead of their sum; the tables' group data are read
// through L1.
struct DpTable {
  MilpDims d;
  int step, n_groups, phases, pad;
  const Group* groups;
  const int* members;
  const double* h;
  const long long* off;
  const unsigned long long* order;
  double* best;
  int* choice;
};
constexpr int kDpMaxTables = 64;

__global__ void __launch_bounds__(256) k4_dp_multi(const DpTable* __restrict__ tabs, int K, int max_phases) {
  __shared__ long long pre[kDpMaxTables + 1];
  __shared__ long long beg[kDpMaxTables];
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (int ph = 0; ph < max_phases; ++ph) {
    if (threadIdx.x < K) {
      const DpTable& T = tabs[threadIdx.x];
      const int l0 = ph * T.step;
      long long b = 0, c = 0;
      if (l0 < T.d.levels) {
        const int l1 = min(l0 + T.step, T.d.levels);
        b = T.off[l0];
        c = T.off[l1] - b;
      }
      beg[threadIdx.x] = b;
      pre[threadIdx.x + 1] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      pre[0] = 0;
      for (int t = 0; t < K; ++t) pre[t + 1] += pre[t];
    }
    __syncthreads();
    const long long total = pre[K];
    for (long long w = warp; w < total; w += n_warps) {
      int lo = 0, hi = K - 1;  // table of work item w: last t with pre[t] <= w
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pre[mid] <= w) lo = mid;
        else hi = mid - 1;
      }
      const DpTable& T = tabs[lo];
      const unsigned long long pk = T.order[beg[lo] + (w - pre[lo])];
      long long s = 0;
      for (int t = 0; t < T.d.T; ++t) s += (long long)((pk >> T.d.off[t]) & T.d.mask[t]) * T.d.stride[t];
      double m = 0.0;
      int ch = -1;
      for (int g = lane; g < T.n_groups; g += 32) {
        const Group G = T.groups[g];
        if ((int)((pk >> T.d.off[G.type]) & T.d.mask[G.type]) < G.n) continue;
        const double bp = T.best[s - G.delta];
        const double v = bp + G.hmax;
        if (v < m) continue;
        int c = INT_MAX;
        for (int k = 0; k < G.count; ++k) {
          const int cc = T.members[G.first + k];
          if (bp + T.h[cc] == v) {
            c = cc;
            break;
          }
        }
        if (v > m) {
          m = v;
          ch = c;
        } else if (c < ch) {
          ch = c;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const int c2 = __shfl_xor_sync(0xffffffffu, ch, o);
        if (m2 > m || (m2 == m && c2 < ch)) {
          m = m2;
          ch = c2;
        }
      }
      if (lane == 0) {
        T.best[s] = m;
        T.choice[s] = ch;
      }
    }
    grid.sync();
  }
}

struct MilpOut {
  double aggregate;
  double makespan;
  int n_entries;
  int pad;
};

// Backtracking + plan assembly, one thread per query (src/rollout_milp.cpp:145-170).
__global__ void k4_backtrack(MilpDims d, int q, const long long* __restrict__ full_idx,
                             const gp_config* __restrict__ cfg, int n_cfg, const double* __restrict__ best,
                             const int* __restrict__ choice, const double* __restrict__ Bs, double len,
                             int* __restrict__ counts_all, gp_rollout_entry* __restrict__ entries_all,
                             MilpOut* __restrict__ outs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= q) return;
  const long long full = full_idx[i];
  const double B = Bs[i];
  int* counts = counts_all + (size_t)i * n_cfg;
  gp_rollout_entry* entries = entries_all + (size_t)i * n_cfg;
  MilpOut* out = outs + i;
  const double agg = best[full];
  out->aggregate = agg;
  out->n_entries = -1;
  if (agg <= 0) return;
  for (int c = 0; c < n_cfg; ++c) counts[c] = 0;
  long long cur = full;
  while (choice[cur] >= 0) {
    const int c = choice[cur];
    counts[c]++;
    for (int t = 0; t < d.T; ++t) cur -= (long long)cfg[c].type_counts[t] * d.stride[t];
  }
  out->makespan = B * len / agg;
  int ne = 0;
  for (int c = 0; c < n_cfg; ++c) {
    if (counts[c] == 0) continue;
    entries[ne].config = c;
    entries[ne].replicas = counts[c];
    entries[ne].workload = B * counts[c] * cfg[c].throughput / agg;
    ++ne;
  }
  out->n_entries = ne;
}

// ------------------------------------------------------------ K6 weight sync
// For each rollout entry type: max link from any train device into any rollout
// device of that type; bottleneck = min over entries (src/cost_model.cpp:174-196).
__global__ void k6_type_maxlink(const int* __restrict__ train, int nt, const int* __restrict__ roll,
                                int nr, const int* __restrict__ dtype, const double* __restrict__ links,
                                int N, double* __restrict__ type_max /* [T] */) {
  const int t = blockIdx.x;
  double m = 0;
  const long long tot = (long long)nt * nr;
  for (long long p = threadIdx.x; p < tot; p += blockDim.x) {
    const int i = (int)(p / nr), j = (int)(p - (long long)i * nr);
    const int di = roll[j];
    if (dtype[di] != t) continue;
    const double l = links[(size_t)train[i] * N + di];
    m = m < l ? l : m;
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, m, o);
    m = m < x ? x : m;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = m < red[w] ? red[w] : m;
    type_max[t] = m;
  }
}

__global__ void k6_combine(const double* __restrict__ type_max, const int* __restrict__ etype,
                           const int* __restrict__ erep, int ne, int window, double mbi,
                           double sync_latency, double* __restrict__ out) {
  double bottleneck = kInf;
  for (int e = 0; e < ne; ++e) {
    if (erep[e] < 1) continue;
    const double best = etype[e] >= 0 ? type_max[etype[e]] : 0.0;
    if (best > 0) bottleneck = best < bottleneck ? best : bottleneck;
  }
  double transfer = 0;
  if (bottleneck < kInf && mbi > 0) transfer = mbi / bottleneck;
  *out = window * transfer + sync_latency;
}

// Batched weight sync: block (set, type) -> max link train(set) x rollout(set, type);
// then one thread per set combines its entries (bottleneck, window transfer + latency).
__global__ void k6_batch_maxlink(const int* __restrict__ ids, const int* __restrict__ t_off,
                                 const int* __restrict__ r_off, int T, const int* __restrict__ dtype,
                                 const double* __restrict__ links, int N, double* __restrict__ type_max) {
  const int set = blockIdx.x / T, t = blockIdx.x % T;
  const int* train = ids + t_off[set];
  const int nt = r_off[set] - t_off[set];
  const int* roll = ids + r_off[set];
  const int nr = t_off[set + 1] - r_off[set];
  double m = 0;
  const long long tot = (long long)nt * nr;
  for (long long p = threadIdx.x; p < tot; p += blockDim.x) {
    const int i = (int)(p / nr), j = (int)(p - (long long)i * nr);
    const int di = roll[j];
    if (dtype[di] != t) continue;
    const double l = links[(size_t)train[i] * N + di];
    m = m < l ? l : m;
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, m, o);
    m = m < x ? x : m;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = m < red[w] ? red[w] : m;
    type_max[blockIdx.x] = m;
  }
}

__global__ void k6_batch_combine(int q, int T, const double* __restrict__ type_max, const int* __restrict__ e_off,
                                 const int* __restrict__ etype, const int* __restrict__ erep, int window,
                                 double mbi, double sync_latency, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= q) return;
  double bottleneck = kInf;
  for (int e = e_off[i]; e < e_off[i + 1]; ++e) {
    if (erep[e] < 1) continue;
    const double best = etype[e] >= 0 ? type_max[(size_t)i * T + etype[e]] : 0.0;
    if (best > 0) bottleneck = best < bottleneck ? best : bottleneck;
  }
  double transfer = 0;
  if (bottleneck < kInf && mbi > 0) transfer = mbi / bottleneck;
  out[i] = window * transfer + sync_latency;
}

// ===================================================================== host

template <typename T>
static T* carve2(char*& p, size_t count) {
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
  T* r = reinterpret_cast<T*>(p);
  p += sizeof(T) * count;
  return r;
}

int rollout_capacities(gp_ctx* ctx, const int32_t* ids, int n, int32_t* caps) {
  for (int t = 0; t < ctx->T; ++t) caps[t] = 0;
  for (int i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= ctx->N) return set_error(GP_INVALID, "unknown device id " + std::to_string(ids[i]));
    caps[ctx->h_type[ids[i]]]++;
  }
  return GP_OK;
}

// enumerate_configs (src/rollout_milp.cpp:39-89), batched over rollout sets: the
// host derives each set's per-type machine availability (enumeration metadata), one
// K3 launch scores every (set, type, TP multiset) candidate, one copy brings them back.
int configs_batch(gp_ctx* ctx, int q, const int32_t* const* ids, const int32_t* ns, const gp_rollout_opts* o,
                  std::vector<std::vector<gp_config>>& out, std::vector<int>* uniq_out) {
  out.assign(q, {});
  if (o->max_stages < 0 || o->max_stages > GP_MAX_ROLLOUT_STAGES)
    return set_error(GP_INVALID, "rollout max_stages must lie in [0, " + std::to_string(GP_MAX_ROLLOUT_STAGES) +
                                     "] (gp_config holds GP_MAX_ROLLOUT_STAGES stages)");
  const int T = ctx->T;
  // The configuration list of a set depends only on its per-type machine availability
  // (the kAv largest per-machine device counts and the machine count of each type), so
  // sets are deduplicated on that signature and K3 runs once per distinct signature.
  std::vector<int> avail, nm;
  std::vector<int> uniq_of(q, -1);
  std::map<std::vector<int>, int> sig_index;
  std::vector<CfgCand> cands;
  std::vector<int> per_machine(ctx->M, 0), mtype(ctx->M, -1);
  std::vector<char> seen(ctx->N, 0);
  constexpr int SW = kAv + 1;
  std::vector<int> sig((size_t)T * SW);
  for (int si = 0; si < q; ++si) {
    const int32_t* id = ids[si];
    const int n = ns[si];
    if (n <= 0) return set_error(GP_INVALID, "enumerate_configs requires a non-empty rollout set");
    std::fill(per_machine.begin(), per_machine.end(), 0);
    for (int i = 0; i < n; ++i) {
      if (id[i] < 0 || id[i] >= ctx->N) return set_error(GP_INVALID, "unknown device id " + std::to_string(id[i]));
      if (seen[id[i]]) {
        for (int j = 0; j < i; ++j) seen[id[j]] = 0;
        return set_error(GP_INVALID, "duplicate device id " + std::to_string(id[i]));
      }
      seen[id[i]] = 1;
      per_machine[ctx->h_machine[id[i]]]++;
      mtype[ctx->h_machine[id[i]]] = ctx->h_type[id[i]];  // machines are type-pure (loader)
    }
    for (int i = 0; i < n; ++i) seen[id[i]] = 0;
    std::vector<std::vector<int>> by_type(T);
    for (int m = 0; m < ctx->M; ++m)
      if (per_machine[m]) by_type[mtype[m]].push_back(per_machine[m]);
    std::fill(sig.begin(), sig.end(), 0);
    for (int t = 0; t < T; ++t) {
      auto& v = by_type[t];
      std::sort(v.rbegin(), v.rend());
      sig[(size_t)t * SW] = (int)v.size();
      for (int k = 0; k < kAv && k < (int)v.size(); ++k) sig[(size_t)t * SW + 1 + k] = v[k];
    }
    auto ins = sig_index.emplace(sig, (int)sig_index.size());
    uniq_of[si] = ins.first->second;
    if (!ins.second) continue;
    const int ui = ins.first->second;
    for (int t = 0; t < T; ++t) {
      nm.push_back(sig[(size_t)t * SW]);
      for (int k = 0; k < kAv; ++k) avail.push_back(sig[(size_t)t * SW + 1 + k]);
      if (by_type[t].empty()) continue;
      // candidates in reference order: stages, then tp_multisets over {8,4,2,1}
      for (int S = 1; S <= o->max_stages; ++S) {
        int tp[kAv];
        std::function<void(int, int)> rec = [&](int d, int mx) {
          if (d == S) {
            CfgCand c{t, S, {}, ui};
            for (int u = 0; u < S; ++u) c.tp[u] = tp[u];
            cands.push_back(c);
            return;
          }
          for (int v2 : {8, 4, 2, 1}) {
            if (v2 > mx) continue;
            tp[d] = v2;
            rec(d + 1, v2);
          }
        };
        rec(0, 8);
      }
    }
  }
  const int nc = (int)cands.size();
  if (nc == 0) {
    if (uniq_out) *uniq_out = std::move(uniq_of);
    return GP_OK;
  }
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += ((b + 255) & ~size_t(255)) + 256; };
  add(sizeof(CfgCand) * nc);
  add(sizeof(int) * avail.size());
  add(sizeof(int) * nm.size());
  add(sizeof(gp_config) * nc);
  add(sizeof(int) * nc);
  char* base = static_cast<char*>(ctx_scratch(ctx, bytes, kArenaRollout));
  if (!base) return GP_CUDA_ERROR;
  char* p = base;
  CfgCand* d_c = carve2<CfgCand>(p, nc);
  int* d_av = carve2<int>(p, avail.size());
  int* d_nm = carve2<int>(p, nm.size());
  gp_config* d_out = carve2<gp_config>(p, nc);
  int* d_keep = carve2<int>(p, nc);
  const size_t in_bytes = (size_t)((char*)(d_nm + nm.size()) - (char*)d_c);
  const size_t out_bytes = (size_t)((char*)(d_keep + nc) - (char*)d_out);
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  char* hp = static_cast<char*>(ctx_pinned(ctx, std::max(in_bytes, out_bytes) + 512));
  if (!hp) return GP_CUDA_ERROR;
  std::memcpy(hp, cands.data(), sizeof(CfgCand) * nc);
  std::memcpy(hp + ((char*)d_av - (char*)d_c), avail.data(), sizeof(int) * avail.size());
  std::memcpy(hp + ((char*)d_nm - (char*)d_c), nm.data(), sizeof(int) * nm.size());
  GP_CUDA(cudaMemcpyAsync(d_c, hp, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += (long long)in_bytes;
  k3_configs<<<(nc + 127) / 128, 128, 0, ctx->stream>>>(d_c, nc, d_av, d_nm, o->max_stages, ctx->sc, ctx->d_tcap,
                                                      ctx->d_thbm, ctx->d_tflops, ctx->d_ceff, ctx->d_ioeff, T,
                                                      d_out, d_keep);
  ctx->launches++;
  GP_CUDA(cudaGetLastError());
  GP_CUDA(cudaMemcpyAsync(hp, d_out, out_bytes, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->d2h_bytes += (long long)out_bytes;
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  const gp_config* h_cfg = reinterpret_cast<const gp_config*>(hp);
  const int* h_keep = reinterpret_cast<const int*>(hp + ((char*)d_keep - (char*)d_out));
  std::vector<std::vector<gp_config>> uniq(sig_index.size());
  for (int i = 0; i < nc; ++i)
    if (h_keep[i]) uniq[cands[i].set].push_back(h_cfg[i]);
  for (int si = 0; si < q; ++si) out[si] = uniq[uniq_of[si]];
  if (uniq_out) *uniq_out = std::move(uniq_of);
  return GP_OK;
}

int rollout_configs(gp_ctx* ctx, const int32_t* ids, int n, const gp_rollout_opts* o, gp_config* out,
                    int cap, int* n_out) {
  *n_out = 0;
  if (n <= 0) return set_error(GP_INVALID, "enumerate_configs requires a non-empty rollout set");
  std::vector<std::vector<gp_config>> res;
  int rc = configs_batch(ctx, 1, &ids, &n, o, res, nullptr);
  if (rc) return rc;
  const int k = (int)res[0].size();
  for (int i = 0; i < k && i < cap; ++i) out[i] = res[0][i];
  *n_out = k;
  if (k > cap) return set_error(GP_CAPACITY, "config buffer too small (" + std::to_string(k) + " needed)");
  return GP_OK;
}

// solve_milp (src/rollout_milp.cpp:91-171)
//
// Lattice tables are cached per configuration list: best[s] and choice[s] depend only
// on the state's coordinates and the configs (the recurrence never looks at the
// capacities except as the lattice bound), so a table computed on a lattice that
// contains the requested one answers it bit-identically. The scheduler solves many
// MILPs with the same configs (rollout sets whose per-type machine availability
// agrees); each is then a backtrack from its own full state.
struct MilpTable {
  std::vector<unsigned char> sig;  // configs + dims
  unsigned long long sig_hash = 0;  // FNV-1a of sig (compared before the bytes)
  MilpDims d{};
  void* buf = nullptr;  // best | choice | order | level offsets/hist/cursor | groups | members | h
  size_t bytes = 0;
  double* best = nullptr;
  int* choice = nullptr;
  unsigned long long* order = nullptr;
  long long* off = nullptr;
  Group* groups = nullptr;
  int* members = nullptr;
  double* h = nullptr;
  int ng = 0, step = 1;
  long long last_use = 0;
  long long pin = -1;  // milp batch epoch that uses it (not evictable within that batch)
  long long pending_epoch = -1;  // batch whose DP launch will (re)compute it
  ~MilpTable() {
    if (buf) cudaFree(buf);
  }
};

// Lattice tables stay resident (B200: 180 GB HBM) up to kMilpCacheBytes, LRU beyond.
constexpr size_t kMilpCacheBytes = (size_t)8 << 30;
static const int kMilpCacheTables = 64;
constexpr size_t kMilpPoolWarm = (size_t)2 << 30;
struct MilpCache {
  std::vector<std::unique_ptr<MilpTable>> tables;
  long long clock = 0, epoch = 0;
  size_t bytes = 0;
  bool pool_ready = false;
};

// GPLAN_PROFILE=1: lattice tables built / reused, states tabulated, DP and backtrack wall time
struct MilpStats {  // (updated from the per-device threads of milp_batch: atomics)
  std::atomic<long long> built{0}, reused{0}, states{0}, backtracks{0}, queries{0}, mallocs{0};
  AtomicD dp_s, bt_s, malloc_s, prep_s, kern_s, sig_s, plan_s;
  std::atomic<long long> levels{0}, groups{0};
  ~MilpStats() {
    if (std::getenv("GPLAN_PROFILE"))
      std::fprintf(stderr,
                   "milp: %lld tables built (%lld states, %lld mallocs, %.3f s), %lld reused, %lld backtrack "
                   "launches for %lld queries (%.3f s); malloc %.3f s, level sort %.3f s, dp kernel %.3f s, "
                   "%lld levels, %lld groups; signatures %.3f s, table planning %.3f s\n",
                   built.load(), states.load(), mallocs.load(), (double)dp_s, reused.load(), backtracks.load(),
                   queries.load(), (double)bt_s, (double)malloc_s, (double)prep_s, (double)kern_s, levels.load(),
                   groups.load(), (double)sig_s, (double)plan_s);
  }
} g_milp_stats;

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void milp_cache_free(gp_ctx* ctx) {
  delete static_cast<MilpCache*>(ctx->milp_cache);
  ctx->milp_cache = nullptr;
}

static void set_dims(MilpDims& d, int dims, const int* caps) {
  d.T = dims;
  long long states = 1;
  int levels = 1, off = 0;
  for (int t = 0; t < dims; ++t) {
    d.stride[t] = states;
    d.cap[t] = caps[t];
    states *= caps[t] + 1;
    levels += caps[t];
    int bits = 1;
    while ((1 << bits) <= caps[t]) ++bits;
    d.off[t] = off;
    d.mask[t] = (1u << bits) - 1u;
    off += bits;
  }
  d.states = states;
  d.levels = levels;
}

static unsigned long long sig_hash(const std::vector<unsigned char>& v) {
  unsigned long long h = 1469598103934665603ULL;
  for (unsigned char c : v) h = (h ^ c) * 1099511628211ULL;
  return h;
}

// Table key: the configs' fields (not their padding bytes) + dims.
static std::vector<unsigned char> milp_sig(const gp_config* cfg, int nc, int dims) {
  std::vector<unsigned char> sig;
  sig.reserve((size_t)nc * (GP_MAX_TYPES * 4 + 8) + 4);
  auto put = [&](const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    sig.insert(sig.end(), b, b + n);
  };
  for (int c = 0; c < nc; ++c) {
    put(cfg[c].type_counts, sizeof(int32_t) * dims);  // the DP reads counts and throughput only
    put(&cfg[c].throughput, sizeof(double));
  }
  put(&dims, sizeof dims);
  return sig;
}

// Validates configs (type-pure, >= 1 device) and returns the (type, devices) grouping key.
static int milp_groups(const gp_config* cfg, int nc, int dims, std::vector<std::pair<long long, int>>& key) {
  key.clear();
  for (int c = 0; c < nc; ++c) {
    int t = -1, n = 0, used = 0;
    for (int u = 0; u < dims; ++u)
      if (cfg[c].type_counts[u] > 0) {
        if (t < 0) t = u;
        ++used;
        n = cfg[c].type_counts[u];
      }
    if (used != 1 || n <= 0)
      return set_error(GP_INVALID, "solve_milp on the GPU requires type-pure configs using >= 1 device");
    key.push_back({(long long)t * 1000000 + n, c});
  }
  std::stable_sort(key.begin(), key.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  return GP_OK;
}

// A table for `cfg` covering `caps`: a cached one, or a new one whose inputs and level
// ordering are enqueued (its DP then runs in run_pending, batched with the others).
static int plan_table(gp_ctx* ctx, const gp_config* cfg, int nc, int dims, const int* caps, MilpTable** out,
                      bool* pending) {
  *pending = false;
  if (!ctx->milp_cache) ctx->milp_cache = new MilpCache();
  MilpCache& mc = *static_cast<MilpCache*>(ctx->milp_cache);
  const std::vector<unsigned char> sig = milp_sig(cfg, nc, dims);
  const unsigned long long sh = sig_hash(sig);
  MilpTable* same = nullptr;
  for (auto& t : mc.tables) {
    if (t->sig_hash != sh || t->sig != sig) continue;
    bool covers = true;
    for (int u = 0; u < dims && covers; ++u) covers = caps[u] <= t->d.cap[u];
    if (covers) {
      t->last_use = ++mc.clock;
      t->pin = mc.epoch;
      *out = t.get();
      g_milp_stats.reused++;
      return GP_OK;
    }
    same = t.get();  // a same-config table: grown to the union lattice below (its DP reruns
                     // before any backtrack of this batch, so its earlier users stay covered)
  }
  std::vector<std::pair<long long, int>> key;
  int rc = milp_groups(cfg, nc, dims, key);
  if (rc) return rc;
  // lattice to tabulate: the union with a cached table of the same configs when that grows
  // the state count by at most 2x (a union of unlike lattices multiplies states)
  std::vector<int> lat(caps, caps + dims);
  if (same) {
    long long u = 1, own = 1;
    std::vector<int> un(dims);
    for (int t = 0; t < dims; ++t) {
      un[t] = std::max(caps[t], same->d.cap[t]);
      u *= un[t] + 1;
      own *= caps[t] + 1;
    }
    if (u <= 50000000 && u <= 2 * std::max(own, same->d.states)) lat = un;
    else same = nullptr;  // keep the cached table; tabulate this lattice separately
  }
  MilpDims d{};
  set_dims(d, dims, lat.data());
  std::vector<Group> groups;
  std::vector<int> members;
  for (size_t i = 0; i < key.size();) {
    size_t j = i;
    const int t = (int)(key[i].first / 1000000), n = (int)(key[i].first % 1000000);
    Group G{t, n, (long long)n * d.stride[t], cfg[key[i].second].throughput, (int)members.size(), 0};
    while (j < key.size() && key[j].first == key[i].first) {
      members.push_back(key[j].second);
      const double hh = cfg[key[j].second].throughput;
      G.hmax = G.hmax < hh ? hh : G.hmax;
      ++j;
    }
    G.count = (int)(j - i);
    groups.push_back(G);
    i = j;
  }
  const int ng = (int)groups.size();
  if (ng > kMaxGroups) return set_error(GP_INVALID, "too many config groups for the sm_100a kernel");
  int step = INT_MAX;
  for (const Group& G : groups) step = std::min(step, G.n);
  std::vector<double> hs(nc);
  for (int c = 0; c < nc; ++c) hs[c] = cfg[c].throughput;
  size_t need = 0;
  auto add = [&](size_t b) { need += ((b + 255) & ~size_t(255)) + 256; };
  add(sizeof(double) * d.states);
  add(sizeof(int) * d.states);
  add(sizeof(unsigned long long) * d.states);
  add(sizeof(long long) * (d.levels + 1));
  add(sizeof(int) * d.levels);
  add(sizeof(int) * d.levels);
  add(sizeof(int));
  add(sizeof(Group) * ng);
  add(sizeof(int) * nc);
  add(sizeof(double) * nc);
  MilpTable* tab = same;
  if (!tab) {  // recycle the least recently used table outside this batch when over budget
    MilpTable* lru = nullptr;
    if (mc.bytes + need > kMilpCacheBytes || (int)mc.tables.size() >= kMilpCacheTables)
      for (auto& t : mc.tables)
        if (t->pin != mc.epoch && (!lru || t->last_use < lru->last_use)) lru = t.get();
    if (lru) {
      tab = lru;
    } else {
      mc.tables.push_back(std::make_unique<MilpTable>());
      tab = mc.tables.back().get();
    }
    tab->sig = sig;
    tab->sig_hash = sh;
  }
  GP_CUDA(cudaStreamSynchronize(ctx->stream));  // the pinned staging buffer is reused below
  if (!mc.pool_ready) {  // stream-ordered allocations stay in the device pool between tables
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      void* warm = nullptr;  // map the table budget once; later tables sub-allocate from it
      if (cudaMallocAsync(&warm, kMilpPoolWarm, ctx->stream) == cudaSuccess) cudaFreeAsync(warm, ctx->stream);
      else cudaGetLastError();
    }
    mc.pool_ready = true;
  }
  if (need > tab->bytes) {  // grow-only, with headroom: tables of one run vary in size
    if (tab->buf) GP_CUDA(cudaFreeAsync(tab->buf, ctx->stream));
    mc.bytes -= tab->bytes;
    tab->buf = nullptr;
    tab->bytes = 0;
    const double t0 = now_s();
    const size_t want = std::max(need + need / 2, (size_t)1 << 20);
    GP_CUDA(cudaMallocAsync(&tab->buf, want, ctx->stream));
    tab->bytes = want;
    mc.bytes += want;
    g_milp_stats.mallocs++;
    g_milp_stats.malloc_s += now_s() - t0;
  }
  char* p = static_cast<char*>(tab->buf);
  tab->best = carve2<double>(p, d.states);
  tab->choice = carve2<int>(p, d.states);
  tab->order = carve2<unsigned long long>(p, d.states);
  tab->off = carve2<long long>(p, d.levels + 1);
  int* d_hist = carve2<int>(p, d.levels);
  int* d_cursor = carve2<int>(p, d.levels);
  int* d_maxw = carve2<int>(p, 1);
  tab->groups = carve2<Group>(p, ng);
  tab->members = carve2<int>(p, nc);
  tab->h = carve2<double>(p, nc);
  const size_t in_bytes = (size_t)((char*)(tab->h + nc) - (char*)tab->groups);
  char* hp = static_cast<char*>(ctx_pinned(ctx, std::max(in_bytes, (size_t)4096)));
  if (!hp) return GP_CUDA_ERROR;
  std::memcpy(hp, groups.data(), sizeof(Group) * ng);
  std::memcpy(hp + ((char*)tab->members - (char*)tab->groups), members.data(), sizeof(int) * nc);
  std::memcpy(hp + ((char*)tab->h - (char*)tab->groups), hs.data(), sizeof(double) * nc);
  GP_CUDA(cudaMemcpyAsync(tab->groups, hp, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += (long long)in_bytes;
  GP_CUDA(cudaMemsetAsync(d_hist, 0, sizeof(int) * d.levels, ctx->stream));
  const int sweep_blocks = (int)std::min<long long>((d.states + 255) / 256, (long long)ctx->num_sms * 16);
  k4_level_hist<<<sweep_blocks, 256, 0, ctx->stream>>>(d, d_hist);
  k4_level_scan<<<1, 32, 0, ctx->stream>>>(d_hist, d.levels, tab->off, d_cursor, d_maxw);
  k4_level_scatter<<<sweep_blocks, 256, 0, ctx->stream>>>(d, tab->off, d_cursor, tab->order);
  ctx->launches += 3;
  tab->d = d;
  tab->ng = ng;
  tab->step = step;
  tab->last_use = ++mc.clock;
  tab->pin = mc.epoch;
  *out = tab;
  *pending = tab->pending_epoch != mc.epoch;  // listed once per batch
  tab->pending_epoch = mc.epoch;
  g_milp_stats.built++;
  g_milp_stats.states += d.states;
  g_milp_stats.levels += d.levels;
  g_milp_stats.groups += ng;
  return GP_OK;
}

// The lattice DPs of the planned tables, kDpMaxTables per cooperative launch.
static int run_pending(gp_ctx* ctx, const std::vector<MilpTable*>& pend) {
  if (pend.empty()) return GP_OK;
  const double t0 = now_s();
  static std::once_flag occ_once;  // (run_pending is called from the per-device threads)
  static int occ = 1;
  std::call_once(occ_once, [] {
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k4_dp_multi, 256, 0);
    occ = std::max(1, o);
  });
  for (size_t c0 = 0; c0 < pend.size(); c0 += kDpMaxTables) {
    const int K = (int)std::min<size_t>(kDpMaxTables, pend.size() - c0);
    std::vector<DpTable> dt(K);
    int max_phases = 0;
    long long max_width = 1;
    for (int k = 0; k < K; ++k) {
      const MilpTable* t = pend[c0 + k];
      DpTable& e = dt[k];
      e.d = t->d;
      e.step = t->step;
      e.n_groups = t->ng;
      e.phases = (t->d.levels + t->step - 1) / t->step;
      e.pad = 0;
      e.groups = t->groups;
      e.members = t->members;
      e.h = t->h;
      e.off = t->off;
      e.order = t->order;
      e.best = t->best;
      e.choice = t->choice;
      max_phases = std::max(max_phases, e.phases);
      max_width += 2 * ((t->d.states + e.phases - 1) / e.phases);
    }
    DpTable* d_dt = static_cast<DpTable*>(ctx_scratch(ctx, sizeof(DpTable) * K, kArenaRollout));
    if (!d_dt) return GP_CUDA_ERROR;
    GP_CUDA(cudaStreamSynchronize(ctx->stream));  // pinned staging + scratch reuse
    char* hp = static_cast<char*>(ctx_pinned(ctx, sizeof(DpTable) * K + 256));
    if (!hp) return GP_CUDA_ERROR;
    std::memcpy(hp, dt.data(), sizeof(DpTable) * K);
    GP_CUDA(cudaMemcpyAsync(d_dt, hp, sizeof(DpTable) * K, cudaMemcpyHostToDevice, ctx->stream));
    ctx->h2d_bytes += (long long)(sizeof(DpTable) * K);
    // grid: about one warp per state of the widest phase sum, at most what is co-resident
    int blocks = (int)std::min<long long>((long long)ctx->num_sms * occ, (max_width + 7) / 8);
    blocks = std::max(1, blocks);
    int K_arg = K;
    void* args[] = {&d_dt, &K_arg, &max_phases};
    GP_CUDA(cudaLaunchCooperativeKernel((void*)k4_dp_multi, blocks, 256, args, 0, ctx->stream));
    ctx->launches++;
  }
  if (std::getenv("GPLAN_PROFILE")) {
    cudaStreamSynchronize(ctx->stream);
    g_milp_stats.kern_s += now_s() - t0;
  }
  return GP_OK;
}

static int ensure_table(gp_ctx* ctx, const gp_config* cfg, int nc, int dims, const int* caps, MilpTable** out) {
  if (!ctx->milp_cache) ctx->milp_cache = new MilpCache();
  static_cast<MilpCache*>(ctx->milp_cache)->epoch++;
  bool pending = false;
  int rc = plan_table(ctx, cfg, nc, dims, caps, out, &pending);
  if (rc) return rc;
  if (pending) rc = run_pending(ctx, {*out});
  return rc;
}

// Backtracks q queries (caps, B, len) of the same configs from `tab` in one launch.
static int backtrack_many(gp_ctx* ctx, MilpTable* tab, const gp_config* cfg, int nc, int q,
                          const int* const* caps, const double* Bs, double len, gp_rollout_result* outs,
                          gp_rollout_entry* const* entries) {
  const double t_start = now_s();
  g_milp_stats.backtracks++;
  g_milp_stats.queries += q;
  std::vector<long long> full(q);
  std::vector<double> Bv(Bs, Bs + q);
  for (int i = 0; i < q; ++i) {
    full[i] = 0;
    for (int t = 0; t < tab->d.T; ++t) full[i] += (long long)caps[i][t] * tab->d.stride[t];
  }
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += ((b + 255) & ~size_t(255)) + 256; };
  add(sizeof(gp_config) * nc);
  add(sizeof(long long) * q);
  add(sizeof(double) * q);
  add(sizeof(int) * (size_t)nc * q);
  add(sizeof(gp_rollout_entry) * (size_t)nc * q);
  add(sizeof(MilpOut) * q);
  char* base = static_cast<char*>(ctx_scratch(ctx, bytes, kArenaMisc));
  if (!base) return GP_CUDA_ERROR;
  char* p = base;
  gp_config* d_cfg = carve2<gp_config>(p, nc);
  long long* d_full = carve2<long long>(p, q);
  double* d_B = carve2<double>(p, q);
  int* d_counts = carve2<int>(p, (size_t)nc * q);
  gp_rollout_entry* d_entries = carve2<gp_rollout_entry>(p, (size_t)nc * q);
  MilpOut* d_mo = carve2<MilpOut>(p, q);
  const size_t in_bytes = (size_t)((char*)(d_B + q) - (char*)d_cfg);
  const size_t out_bytes = (size_t)((char*)(d_mo + q) - (char*)d_entries);
  char* hp = static_cast<char*>(ctx_pinned(ctx, std::max(in_bytes, out_bytes) + 512));
  if (!hp) return GP_CUDA_ERROR;
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(hp, cfg, sizeof(gp_config) * nc);
  std::memcpy(hp + ((char*)d_full - (char*)d_cfg), full.data(), sizeof(long long) * q);
  std::memcpy(hp + ((char*)d_B - (char*)d_cfg), Bv.data(), sizeof(double) * q);
  GP_CUDA(cudaMemcpyAsync(d_cfg, hp, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += (long long)in_bytes;
  k4_backtrack<<<(q + 31) / 32, 32, 0, ctx->stream>>>(tab->d, q, d_full, d_cfg, nc, tab->best, tab->choice, d_B,
                                                     len, d_counts, d_entries, d_mo);
  ctx->launches++;
  GP_CUDA(cudaGetLastError());
  GP_CUDA(cudaMemcpyAsync(hp, d_entries, out_bytes, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->d2h_bytes += (long long)out_bytes;
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  const gp_rollout_entry* he = reinterpret_cast<const gp_rollout_entry*>(hp);
  const MilpOut* ho = reinterpret_cast<const MilpOut*>(hp + ((char*)d_mo - (char*)d_entries));
  for (int i = 0; i < q; ++i) {
    gp_rollout_result& o = outs[i];
    std::memset(&o, 0, sizeof o);
    o.total_rollouts = Bs[i];
    o.aggregate = ho[i].aggregate;
    long long states = 1;
    for (int t = 0; t < tab->d.T; ++t) states *= caps[i][t] + 1;
    o.states = states;
    o.n_entries = ho[i].n_entries;  // -1: infeasible (aggregate <= 0)
    if (ho[i].n_entries >= 0) {
      o.makespan = ho[i].makespan;
      std::memcpy(entries[i], he + (size_t)nc * i, sizeof(gp_rollout_entry) * ho[i].n_entries);
    }
  }
  g_milp_stats.bt_s += now_s() - t_start;
  return GP_OK;
}

static int milp_check(int nc, const int32_t* caps, int dims) {
  if (dims < 1 || dims > GP_MAX_TYPES) return set_error(GP_INVALID, "dims must lie in [1, GP_MAX_TYPES]");
  if (nc > kMaxCfg) return set_error(GP_INVALID, "too many replica configurations for the sm_100a kernel");
  long long states = 1;
  for (int t = 0; t < dims; ++t) {
    if (caps[t] < 0) return set_error(GP_INVALID, "negative capacity");
    states *= caps[t] + 1;
    if (states > 50000000) return set_error(GP_INVALID, "capacity lattice too large for the exact solver");
  }
  return GP_OK;
}

int solve_milp(gp_ctx* ctx, const gp_config* cfg, int nc, const int32_t* caps, int dims, double B,
               double len, gp_rollout_result* out, gp_rollout_entry* entries) {
  std::memset(out, 0, sizeof *out);
  out->total_rollouts = B;
  if (B <= 0) return GP_OK;
  if (nc == 0) return set_error(GP_INFEASIBLE, "no replica configuration available");
  int rc = milp_check(nc, caps, dims);
  if (rc) return rc;
  MilpTable* tab = nullptr;
  rc = ensure_table(ctx, cfg, nc, dims, caps, &tab);
  if (rc) return rc;
  const int* cp = caps;
  rc = backtrack_many(ctx, tab, cfg, nc, 1, &cp, &B, len, out, &entries);
  if (rc) return rc;
  if (out->n_entries < 0) {
    out->n_entries = 0;
    return set_error(GP_INFEASIBLE, "rollout capacity cannot host any replica");
  }
  return GP_OK;
}

// Many MILPs (one scheduler evaluation batch). Results per query: GP_OK with a plan,
// GP_INFEASIBLE (no configs / aggregate <= 0), or GP_INVALID (lattice > 5e7) in rcs[i].
static int milp_batch_one(gp_ctx* ctx, int q, const gp_config* const* cfgs, const int* ncs,
                          const int32_t* const* caps, int dims, const double* Bs, double len,
                          gp_rollout_result* outs, gp_rollout_entry* const* entries, int* rcs) {
  // group queries with identical config lists
  const double t_sig = now_s();
  std::vector<int> order(q);
  std::vector<std::vector<unsigned char>> sigs(q);
  for (int i = 0; i < q; ++i) {
    order[i] = i;
    sigs[i] = milp_sig(cfgs[i], ncs[i], dims);
    std::memset(&outs[i], 0, sizeof outs[i]);
    outs[i].total_rollouts = Bs[i];
    rcs[i] = GP_OK;
    if (Bs[i] <= 0) { rcs[i] = -1; continue; }  // empty plan
    if (ncs[i] == 0) { rcs[i] = GP_INFEASIBLE; continue; }
    if (milp_check(ncs[i], caps[i], dims)) rcs[i] = GP_INVALID;
  }
  std::vector<unsigned long long> hs(q);
  for (int i = 0; i < q; ++i) hs[i] = sig_hash(sigs[i]);
  // group equal config lists (hash first; the grouping order only decides table planning order)
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return hs[a] != hs[b] ? hs[a] < hs[b] : sigs[a] < sigs[b]; });
  std::vector<std::vector<int>> all_parts;  // queries per table, over all config lists
  std::vector<std::vector<int>> all_caps;   // each table's lattice
  for (size_t g0 = 0; g0 < order.size();) {
    size_t g1 = g0;
    while (g1 < order.size() && hs[order[g1]] == hs[order[g0]] && sigs[order[g1]] == sigs[order[g0]]) ++g1;
    std::vector<int> live;
    for (size_t j = g0; j < g1; ++j)
      if (rcs[order[j]] == GP_OK) live.push_back(order[j]);
    if (!live.empty()) {
      // largest lattices first: each later query whose capacities are covered by an
      // already tabulated lattice of the group is answered from that table
      std::sort(live.begin(), live.end(), [&](int a, int b) {
        long long sa = 1, sb = 1;
        for (int t = 0; t < dims; ++t) {
          sa *= caps[a][t] + 1;
          sb *= caps[b][t] + 1;
        }
        return sa > sb || (sa == sb && a < b);
      });
      std::vector<std::vector<int>> parts;      // queries per table
      std::vector<std::vector<int>> part_caps;  // the table's lattice
      for (int i : live) {
        int hit = -1;
        for (size_t pidx = 0; pidx < parts.size() && hit < 0; ++pidx) {
          bool cov = true;
          for (int t = 0; t < dims && cov; ++t) cov = caps[i][t] <= part_caps[pidx][t];
          if (cov) hit = (int)pidx;
        }
        if (hit < 0) {
          parts.push_back({});
          part_caps.emplace_back(caps[i], caps[i] + dims);
          hit = (int)parts.size() - 1;
        }
        parts[hit].push_back(i);
      }
      for (size_t pidx = 0; pidx < parts.size(); ++pidx) {
        all_parts.push_back(parts[pidx]);
        all_caps.push_back(part_caps[pidx]);
      }
    }
    g0 = g1;
  }
  g_milp_stats.sig_s += now_s() - t_sig;
  // every table of the batch planned first (cached or new), the new ones' DPs batched
  const double t_plan = now_s();
  if (!ctx->milp_cache) ctx->milp_cache = new MilpCache();
  static_cast<MilpCache*>(ctx->milp_cache)->epoch++;
  std::vector<MilpTable*> tabs(all_parts.size()), pend;
  for (size_t pidx = 0; pidx < all_parts.size(); ++pidx) {
    const int i0 = all_parts[pidx][0];
    bool pending = false;
    int rc = plan_table(ctx, cfgs[i0], ncs[i0], dims, all_caps[pidx].data(), &tabs[pidx], &pending);
    if (rc) return rc;
    if (pending) pend.push_back(tabs[pidx]);
  }
  g_milp_stats.plan_s += now_s() - t_plan;
  {
    int rc = run_pending(ctx, pend);
    if (rc) return rc;
  }
  {
    {
      for (size_t pidx = 0; pidx < all_parts.size(); ++pidx) {
        const std::vector<int>& part = all_parts[pidx];
        const int i0 = part[0];
        MilpTable* tab = tabs[pidx];
        int rc = GP_OK;
        std::vector<const int*> cp;
        std::vector<double> bb;
        std::vector<gp_rollout_result> ro(part.size());
        std::vector<gp_rollout_entry*> ep;
        for (int i : part) {
          cp.push_back(caps[i]);
          bb.push_back(Bs[i]);
          ep.push_back(entries[i]);
        }
        rc = backtrack_many(ctx, tab, cfgs[i0], ncs[i0], (int)part.size(), cp.data(), bb.data(), len, ro.data(),
                            ep.data());
        if (rc) return rc;
        for (size_t j = 0; j < part.size(); ++j) {
          outs[part[j]] = ro[j];
          if (ro[j].n_entries < 0) {
            outs[part[j]].n_entries = 0;
            rcs[part[j]] = GP_INFEASIBLE;
          }
        }
      }
    }
  }
  for (int i = 0; i < q; ++i)
    if (rcs[i] == -1) rcs[i] = GP_OK;
  return GP_OK;
}

int weight_sync_batch(gp_ctx* ctx, int q, const int32_t* const* train, const int32_t* nt,
                      const int32_t* const* roll, const int32_t* nr, const int32_t* const* etype,
                      const int32_t* const* erep, const int32_t* ne, int window, double* out) {
  if (q <= 0) return GP_OK;
  const int T = ctx->T;
  std::vector<int> ids, t_off, r_off, e_off, et, er;
  for (int i = 0; i < q; ++i) {
    t_off.push_back((int)ids.size());
    ids.insert(ids.end(), train[i], train[i] + nt[i]);
    r_off.push_back((int)ids.size());
    ids.insert(ids.end(), roll[i], roll[i] + nr[i]);
    e_off.push_back((int)et.size());
    et.insert(et.end(), etype[i], etype[i] + ne[i]);
    er.insert(er.end(), erep[i], erep[i] + ne[i]);
  }
  t_off.push_back((int)ids.size());
  e_off.push_back((int)et.size());
  for (int id : ids)
    if (id < 0 || id >= ctx->N) return set_error(GP_INVALID, "unknown device id");
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += ((b + 255) & ~size_t(255)) + 256; };
  add(sizeof(int) * (ids.size() + 1));
  add(sizeof(int) * t_off.size());
  add(sizeof(int) * r_off.size());
  add(sizeof(int) * e_off.size());
  add(sizeof(int) * (et.size() + 1));
  add(sizeof(int) * (er.size() + 1));
  add(sizeof(double) * (size_t)q * T);
  add(sizeof(double) * q);
  char* base = static_cast<char*>(ctx_scratch(ctx, bytes, kArenaMisc));
  if (!base) return GP_CUDA_ERROR;
  char* p = base;
  int* d_ids = carve2<int>(p, ids.size() + 1);
  int* d_toff = carve2<int>(p, t_off.size());
  int* d_roff = carve2<int>(p, r_off.size());
  int* d_eoff = carve2<int>(p, e_off.size());
  int* d_et = carve2<int>(p, et.size() + 1);
  int* d_er = carve2<int>(p, er.size() + 1);
  double* d_tm = carve2<double>(p, (size_t)q * T);
  double* d_out = carve2<double>(p, q);
  const size_t in_bytes = (size_t)((char*)(d_er + er.size() + 1) - (char*)d_ids);
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  char* hp = static_cast<char*>(ctx_pinned(ctx, std::max(in_bytes, sizeof(double) * q) + 256));
  if (!hp) return GP_CUDA_ERROR;
  auto put = [&](const std::vector<int>& v, void* dptr) {
    if (!v.empty()) std::memcpy(hp + ((char*)dptr - (char*)d_ids), v.data(), sizeof(int) * v.size());
  };
  put(ids, d_ids);
  put(t_off, d_toff);
  put(r_off, d_roff);
  put(e_off, d_eoff);
  put(et, d_et);
  put(er, d_er);
  GP_CUDA(cudaMemcpyAsync(d_ids, hp, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += (long long)in_bytes;
  k6_batch_maxlink<<<q * T, 256, 0, ctx->stream>>>(d_ids, d_toff, d_roff, T, ctx->d_type, ctx->d_links, ctx->N,
                                                   d_tm);
  k6_batch_combine<<<(q + 127) / 128, 128, 0, ctx->stream>>>(q, T, d_tm, d_eoff, d_et, d_er, window, ctx->sc.mbi,
                                                            ctx->sc.sync_latency, d_out);
  ctx->launches += 2;
  GP_CUDA(cudaGetLastError());
  GP_CUDA(cudaMemcpyAsync(hp, d_out, sizeof(double) * q, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->d2h_bytes += (long long)(sizeof(double) * q);
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(out, hp, sizeof(double) * q);
  return GP_OK;
}

int weight_sync(gp_ctx* ctx, const int32_t* train, int nt, const int32_t* roll, int nr,
                const int32_t* etype, const int32_t* erep, int ne, int window, double* out) {
  for (int i = 0; i < nt; ++i)
    if (train[i] < 0 || train[i] >= ctx->N) return set_error(GP_INVALID, "unknown device id");
  for (int i = 0; i < nr; ++i)
    if (roll[i] < 0 || roll[i] >= ctx->N) return set_error(GP_INVALID, "unknown device id");
  const int T = ctx->T;
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += ((b + 255) & ~size_t(255)) + 256; };
  add(sizeof(int) * (nt + 1));
  add(sizeof(int) * (nr + 1));
  add(sizeof(int) * (ne + 1));
  add(sizeof(int) * (ne + 1));
  add(sizeof(double) * T);
  add(sizeof(double));
  char* base = static_cast<char*>(ctx_scratch(ctx, bytes, kArenaRollout));
  if (!base) return GP_CUDA_ERROR;
  char* p = base;
  int* d_t = carve2<int>(p, nt + 1);
  int* d_r = carve2<int>(p, nr + 1);
  int* d_et = carve2<int>(p, ne + 1);
  int* d_er = carve2<int>(p, ne + 1);
  double* d_tm = carve2<double>(p, T);
  double* d_out = carve2<double>(p, 1);
  const size_t in_bytes = (size_t)((char*)(d_er + ne + 1) - (char*)d_t);
  char* hp = static_cast<char*>(ctx_pinned(ctx, std::max(in_bytes, (size_t)64)));
  if (!hp) return GP_CUDA_ERROR;
  std::memcpy(hp, train, sizeof(int) * nt);
  std::memcpy(hp + ((char*)d_r - (char*)d_t), roll, sizeof(int) * nr);
  if (ne) std::memcpy(hp + ((char*)d_et - (char*)d_t), etype, sizeof(int) * ne);
  if (ne) std::memcpy(hp + ((char*)d_er - (char*)d_t), erep, sizeof(int) * ne);
  GP_CUDA(cudaMemcpyAsync(d_t, hp, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += (long long)in_bytes;
  k6_type_maxlink<<<T, 256, 0, ctx->stream>>>(d_t, nt, d_r, nr, ctx->d_type, ctx->d_links, ctx->N, d_tm);
  k6_combine<<<1, 1, 0, ctx->stream>>>(d_tm, d_et, d_er, ne, window, ctx->sc.mbi, ctx->sc.sync_latency,
                                       d_out);
  ctx->launches += 2;
  GP_CUDA(cudaGetLastError());
  double* ho = reinterpret_cast<double*>(hp);
  GP_CUDA(cudaMemcpyAsync(ho, d_out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->d2h_bytes += sizeof(double);
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  *out = *ho;
  return GP_OK;
}

}  // namespace gp

namespace gp {

// Many solve_milp instances (the scheduler's batches). On a multi-device context the queries
// are split by configuration list — every list always goes to the same device, so its cached
// lattice tables stay there across iterations — and the devices run their shares
// concurrently (one host thread each); results land in the caller's arrays in query order.
int milp_batch(gp_ctx* ctx, int q, const gp_config* const* cfgs, const int* ncs, const int32_t* const* caps,
               int dims, const double* Bs, double len, gp_rollout_result* outs, gp_rollout_entry* const* entries,
               int* rcs) {
  const int D = 1 + (int)ctx->peers.size();
  long long states = 0;  // (lattice states of the batch: small batches stay on one device)
  for (int i = 0; i < q && states < kMilpSplitMinStates; ++i) {
    long long st = 1;
    for (int t = 0; t < dims; ++t) st *= caps[i][t] + 1;
    states += st;
  }
  if (D == 1 || q < 2 || states < kMilpSplitMinStates)
    return milp_batch_one(ctx, q, cfgs, ncs, caps, dims, Bs, len, outs, entries, rcs);
  std::vector<std::vector<int>> part(D);
  for (int i = 0; i < q; ++i) {
    const std::vector<unsigned char> sig = milp_sig(cfgs[i], ncs[i], dims);
    unsigned long long h = 1469598103934665603ULL;  // FNV-1a of the configuration list
    for (unsigned char c : sig) h = (h ^ c) * 1099511628211ULL;
    part[h % D].push_back(i);
  }
  std::vector<int> rc_dev(D, GP_OK);
  std::vector<std::string> err(D);
  auto run = [&](int d) {
    const std::vector<int>& pj = part[d];
    if (pj.empty()) return;
    gp_ctx* c = d == 0 ? ctx : ctx->peers[d - 1];
    cudaSetDevice(c->device);
    const int m = (int)pj.size();
    std::vector<const gp_config*> cf(m);
    std::vector<int> nc(m), rc(m);
    std::vector<const int32_t*> cp(m);
    std::vector<double> b(m);
    std::vector<gp_rollout_result> o(m);
    std::vector<gp_rollout_entry*> e(m);
    for (int j = 0; j < m; ++j) {
      cf[j] = cfgs[pj[j]];
      nc[j] = ncs[pj[j]];
      cp[j] = caps[pj[j]];
      b[j] = Bs[pj[j]];
      e[j] = entries[pj[j]];
    }
    rc_dev[d] = milp_batch_one(c, m, cf.data(), nc.data(), cp.data(), dims, b.data(), len, o.data(), e.data(),
                               rc.data());
    if (rc_dev[d]) {
      err[d] = gp_last_error();
      return;
    }
    for (int j = 0; j < m; ++j) {
      outs[pj[j]] = o[j];
      rcs[pj[j]] = rc[j];
    }
  };
  std::vector<std::thread> th;
  for (int d = 1; d < D; ++d) th.emplace_back(run, d);
  run(0);
  for (auto& t : th) t.join();
  cudaSetDevice(ctx->device);
  for (int d = 0; d < D; ++d)
    if (rc_dev[d]) return set_error(rc_dev[d], err[d].empty() ? std::string("milp batch failed") : err[d]);
  return GP_OK;
}

}  // namespace gp
