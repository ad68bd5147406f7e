// exhaustive.cu — the exhaustive rows of SURVEY.md §8f (rank 2), on the GPU:
//   * the product-space training search (enumerate_train_candidates x train_plan_fits x
//     train_step_cost, first minimum; src/train_search.cpp:179-216, tests/oracles.cpp:166-174),
//   * brute_milp_unbounded (tests/oracles.cpp:16-115): every integer replica vector,
//   * exhaustive_schedule_optimum (tests/oracles.cpp:144-209) over every bipartition.
//
// Product space. For a fixed block list the candidates differ only in per-stage (tp, dp);
// fill/drain and transfers do not depend on them and the per-step time is monotone in the
// stage maximum, so the cheapest candidate of a block list reaches max_s min_o total_s(o).
// K2c in mode 1 tabulates min_o total per (block, layers); the layout scan (K1) then returns
// the product-space minimum and the first block list reaching it; k1_finalize decodes the
// first option combination in odometer order that keeps the maximum (per stage the lowest
// tp with total <= M*). Candidate counts / indices come from enumeration metadata
// (train_candidates_meta).
//
// Brute MILP. One thread per rollout set walks the recursion of enumerate_all iteratively
// (same order, same `agg + y * h` accumulation and `theta < best - 1e-15` improvement rule).
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include "gp_internal.h"

namespace gp {

int train_batch(gp_ctx* ctx, int n_sets, const int32_t* const* ids, const int32_t* ns, int window,
                const gp_train_opts* o, gp_train_result* outs, int32_t* const* stage_devices, int mode = 0);
int train_search(gp_ctx* ctx, const int32_t* ids, int n, int window, const gp_train_opts* o,
                 long long lo, long long hi, gp_train_result* out, int32_t* stage_devices, int mode = 0);
int train_candidates_meta(gp_ctx* ctx, const int32_t* ids, int n, const gp_train_result* res,
                          const int32_t* stage_devices, long long* count, long long* index);
int configs_batch(gp_ctx* ctx, int q, const int32_t* const* ids, const int32_t* ns, const gp_rollout_opts* o,
                  std::vector<std::vector<gp_config>>& out, std::vector<int>* uniq_of = nullptr);
int weight_sync_batch(gp_ctx* ctx, int q, const int32_t* const* train, const int32_t* nt,
                      const int32_t* const* roll, const int32_t* nr, const int32_t* const* etype,
                      const int32_t* const* erep, const int32_t* ne, int window, double* out);

constexpr int kBruteMaxCfg = 256;

struct BruteOut {
  double theta;
  long long vectors;
  int feasible;
  int pad;
};

__global__ void __launch_bounds__(128) k7_brute_milp(int q, const gp_config* __restrict__ cfg,
                                                     const int* __restrict__ cfg_off,
                                                     const int* __restrict__ caps, int T,
                                                     const double* __restrict__ Bs, double len,
                                                     int* __restrict__ counts, BruteOut* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= q) return;
  const int off = cfg_off[i], nc = cfg_off[i + 1] - off;
  const gp_config* c = cfg + off;
  const double B = Bs[i];
  for (int j = 0; j < nc; ++j) counts[off + j] = 0;
  BruteOut o{0.0, 0, 0, 0};
  if (B <= 0) {  // tests/oracles.cpp:21-26
    o.feasible = 1;
    out[i] = o;
    return;
  }
  int cap[GP_MAX_TYPES];
  for (int t = 0; t < T; ++t) cap[t] = caps[(size_t)i * T + t];
  int y[kBruteMaxCfg], bnd[kBruteMaxCfg];
  double aggs[kBruteMaxCfg + 1];
  aggs[0] = 0.0;
  int d = 0;
  while (true) {
    if (d == nc) {  // leaf: Rec::go with idx == configs.size()
      ++o.vectors;
      const double agg = aggs[nc];
      if (agg > 0) {
        const double theta = B * len / agg;
        if (!o.feasible || theta < o.theta - 1e-15) {
          o.feasible = 1;
          o.theta = theta;
          for (int j = 0; j < nc; ++j) counts[off + j] = y[j];
        }
      }
      int dd = nc - 1;  // deepest level with another y to try
      while (dd >= 0 && y[dd] >= bnd[dd]) {
        for (int t = 0; t < T; ++t) cap[t] += y[dd] * c[dd].type_counts[t];
        --dd;
      }
      if (dd < 0) break;
      for (int t = 0; t < T; ++t) cap[t] -= c[dd].type_counts[t];
      ++y[dd];
      aggs[dd + 1] = aggs[dd] + y[dd] * c[dd].throughput;
      d = dd + 1;
      continue;
    }
    int bound = INT_MAX;  // level d entered with y = 0 (bound from the remaining capacity)
    bool uses = false;
    for (int t = 0; t < T; ++t) {
      const int v = c[d].type_counts[t];
      if (v > 0) {
        uses = true;
        bound = min(bound, cap[t] / v);
      }
    }
    bnd[d] = uses ? bound : 0;
    y[d] = 0;
    aggs[d + 1] = aggs[d] + 0 * c[d].throughput;
    ++d;
  }
  out[i] = o;
}

// Many brute_milp_unbounded instances in one launch.
int brute_batch(gp_ctx* ctx, int q, const std::vector<const std::vector<gp_config>*>& cfgs,
                const std::vector<const int32_t*>& caps, const std::vector<double>& Bs, double len,
                std::vector<std::vector<int>>& counts, std::vector<BruteOut>& outs) {
  counts.assign(q, {});
  outs.assign(q, BruteOut{});
  if (q <= 0) return GP_OK;
  const int T = ctx->T;
  std::vector<int> off(q + 1, 0);
  for (int i = 0; i < q; ++i) {
    if ((int)cfgs[i]->size() > kBruteMaxCfg) return set_error(GP_INVALID, "brute MILP: too many configs");
    off[i + 1] = off[i] + (int)cfgs[i]->size();
  }
  const int ncfg = off[q];
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += ((b + 255) & ~size_t(255)) + 256; };
  add(sizeof(gp_config) * (ncfg + 1));
  add(sizeof(int) * (q + 1));
  add(sizeof(int) * (size_t)q * T);
  add(sizeof(double) * q);
  add(sizeof(int) * (ncfg + 1));
  add(sizeof(BruteOut) * q);
  char* base = static_cast<char*>(ctx_scratch(ctx, bytes, kArenaMisc));
  if (!base) return GP_CUDA_ERROR;
  auto carve = [](char*& p, size_t b) {
    p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
    char* r = p;
    p += b;
    return r;
  };
  char* p = base;
  gp_config* d_cfg = reinterpret_cast<gp_config*>(carve(p, sizeof(gp_config) * (ncfg + 1)));
  int* d_off = reinterpret_cast<int*>(carve(p, sizeof(int) * (q + 1)));
  int* d_caps = reinterpret_cast<int*>(carve(p, sizeof(int) * (size_t)q * T));
  double* d_B = reinterpret_cast<double*>(carve(p, sizeof(double) * q));
  int* d_counts = reinterpret_cast<int*>(carve(p, sizeof(int) * (ncfg + 1)));
  BruteOut* d_out = reinterpret_cast<BruteOut*>(carve(p, sizeof(BruteOut) * q));
  const size_t in_bytes = (size_t)((char*)(d_B + q) - (char*)d_cfg);
  const size_t out_bytes = (size_t)((char*)(d_out + q) - (char*)d_counts);
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  char* hp = static_cast<char*>(ctx_pinned(ctx, std::max(in_bytes, out_bytes) + 512));
  if (!hp) return GP_CUDA_ERROR;
  for (int i = 0; i < q; ++i)
    if (!cfgs[i]->empty())
      std::memcpy(hp + ((char*)(d_cfg + off[i]) - (char*)d_cfg), cfgs[i]->data(), sizeof(gp_config) * cfgs[i]->size());
  std::memcpy(hp + ((char*)d_off - (char*)d_cfg), off.data(), sizeof(int) * (q + 1));
  for (int i = 0; i < q; ++i)
    std::memcpy(hp + ((char*)(d_caps + (size_t)i * T) - (char*)d_cfg), caps[i], sizeof(int) * T);
  std::memcpy(hp + ((char*)d_B - (char*)d_cfg), Bs.data(), sizeof(double) * q);
  GP_CUDA(cudaMemcpyAsync(d_cfg, hp, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += (long long)in_bytes;
  k7_brute_milp<<<(q + 127) / 128, 128, 0, ctx->stream>>>(q, d_cfg, d_off, d_caps, T, d_B, len, d_counts, d_out);
  ctx->launches++;
  GP_CUDA(cudaGetLastError());
  GP_CUDA(cudaMemcpyAsync(hp, d_counts, out_bytes, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->d2h_bytes += (long long)out_bytes;
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  const int* hc = reinterpret_cast<const int*>(hp);
  const BruteOut* ho = reinterpret_cast<const BruteOut*>(hp + ((char*)d_out - (char*)d_counts));
  for (int i = 0; i < q; ++i) {
    counts[i].assign(hc + off[i], hc + off[i + 1]);
    outs[i] = ho[i];
  }
  return GP_OK;
}

int train_candidates_search(gp_ctx* ctx, const int32_t* ids, int n, int window, gp_train_result* out,
                            int32_t* stage_devices) {
  const gp_train_opts o{4, 16};  // TrainSearchOptions defaults
  int rc = train_search(ctx, ids, n, window, &o, 0, -1, out, stage_devices, 1);
  if (rc) return rc;
  long long count = 0, index = -1;
  rc = train_candidates_meta(ctx, ids, n, out, stage_devices, &count, &index);
  if (rc) return rc;
  out->layouts = count;
  out->feasible = -1;
  if (out->found) out->rank = index;
  return GP_OK;
}

int exhaustive_optimum(gp_ctx* ctx, int window, gp_exhaustive_result* out, int32_t* train_ids) {
  std::memset(out, 0, sizeof *out);
  const int N = ctx->N, T = ctx->T;
  if (N < 2 || N > 20) return set_error(GP_INVALID, "exhaustive optimum: 2 <= devices <= 20");
  const double total_rollouts = static_cast<double>(ctx->work.batch_rollouts) * window;
  const gp_train_opts to{4, 16};
  const gp_rollout_opts ro{4};
  const long long masks = (1LL << N) - 2;
  const int chunk = 8192;
  double ph[5] = {0, 0, 0, 0, 0};  // GPLAN_PROFILE: train, counts, configs, brute, weight sync
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto since = [&](std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(now() - t0).count();
  };
  bool have = false, have_c = false;
  double best = 0, best_c = 0;
  long long best_mask = 0, best_mask_c = 0;
  for (long long m0 = 1; m0 <= masks; m0 += chunk) {
    const int q = (int)std::min<long long>(chunk, masks - m0 + 1);
    std::vector<std::vector<int32_t>> tr(q), rl(q);
    std::vector<const int32_t*> tp(q), rp(q);
    std::vector<int32_t> tn(q), rn(q);
    for (int i = 0; i < q; ++i) {
      const long long mask = m0 + i;
      for (int d = 0; d < N; ++d) ((mask >> d) & 1 ? tr[i] : rl[i]).push_back(d);
      tp[i] = tr[i].data();
      tn[i] = (int32_t)tr[i].size();
      rp[i] = rl[i].data();
      rn[i] = (int32_t)rl[i].size();
    }
    // training side: product-space optimum per train set
    std::vector<gp_train_result> tres(q);
    auto t0 = now();
    int rc = train_batch(ctx, q, tp.data(), tn.data(), window, &to, tres.data(), nullptr, 1);
    if (rc) return rc;
    ph[0] += since(t0);
    t0 = now();
    for (int i = 0; i < q; ++i) {
      long long count = 0, index = 0;
      rc = train_candidates_meta(ctx, tp[i], tn[i], nullptr, nullptr, &count, &index);
      if (rc) return rc;
      out->train_candidates += count;
    }
    // rollout side: configs, brute MILP, weight sync
    ph[1] += since(t0);
    t0 = now();
    std::vector<std::vector<gp_config>> cfgs;
    std::vector<int> cfg_class;
    rc = configs_batch(ctx, q, rp.data(), rn.data(), &ro, cfgs, &cfg_class);
    if (rc) return rc;
    ph[2] += since(t0);
    t0 = now();
    // The brute MILP depends only on (configs, capacities, B): sets sharing a config class
    // and per-type capacities share one solve.
    std::vector<int> live, job_of;
    std::vector<const std::vector<gp_config>*> bc;
    std::vector<std::vector<int32_t>> caps;
    std::vector<const int32_t*> capp;
    std::vector<double> Bs;
    std::map<std::vector<int32_t>, int> job_index;
    for (int i = 0; i < q; ++i) {
      if (!tres[i].found || cfgs[i].empty()) continue;
      live.push_back(i);
    }
    std::vector<int32_t> key(T + 1);
    for (size_t j = 0; j < live.size(); ++j) {
      const int i = live[j];
      std::fill(key.begin(), key.end(), 0);
      key[T] = cfg_class[i];
      for (int d : rl[i]) key[ctx->h_type[d]]++;  // rollout_capacities (src/rollout_milp.cpp:30-37)
      auto ins = job_index.emplace(key, (int)caps.size());
      job_of.push_back(ins.first->second);
      if (!ins.second) continue;
      caps.emplace_back(key.begin(), key.begin() + T);
      bc.push_back(&cfgs[i]);
      Bs.push_back(total_rollouts);
    }
    for (auto& c : caps) capp.push_back(c.data());
    std::vector<std::vector<int>> jcounts;
    std::vector<BruteOut> jbo;
    rc = brute_batch(ctx, (int)caps.size(), bc, capp, Bs, ctx->work.mean_len, jcounts, jbo);
    if (rc) return rc;
    std::vector<const std::vector<int>*> counts(live.size());
    std::vector<BruteOut> bo(live.size());
    for (size_t j = 0; j < live.size(); ++j) {
      counts[j] = &jcounts[job_of[j]];
      bo[j] = jbo[job_of[j]];
    }
    ph[3] += since(t0);
    t0 = now();
    std::vector<int> wl;
    std::vector<const int32_t*> wt, wr, wet, wer;
    std::vector<int32_t> wtn, wrn, wne;
    std::vector<std::vector<int32_t>> et(live.size()), er(live.size());
    for (size_t j = 0; j < live.size(); ++j) {
      out->replica_vectors += bo[j].vectors;
      if (!bo[j].feasible) continue;
      const int i = live[j];
      const std::vector<int>& cj = *counts[j];
      for (size_t c = 0; c < cj.size(); ++c) {
        if (cj[c] <= 0) continue;
        int type = 0;  // ReplicaConfig::gpu_type
        while (type < T && cfgs[i][c].type_counts[type] == 0) ++type;
        et[j].push_back(type);
        er[j].push_back(cj[c]);
      }
      wl.push_back((int)j);
      wt.push_back(tp[i]);
      wtn.push_back(tn[i]);
      wr.push_back(rp[i]);
      wrn.push_back(rn[i]);
      wet.push_back(et[j].data());
      wer.push_back(er[j].data());
      wne.push_back((int32_t)et[j].size());
    }
    std::vector<double> upd(wl.size());
    rc = weight_sync_batch(ctx, (int)wl.size(), wt.data(), wtn.data(), wr.data(), wrn.data(), wet.data(),
                           wer.data(), wne.data(), window, upd.data());
    if (rc) return rc;
    ph[4] += since(t0);
    // selection in mask order (tests/oracles.cpp:196-207)
    for (size_t k = 0; k < wl.size(); ++k) {
      const int j = wl[k], i = live[j];
      const double c_train = tres[i].cost;
      const double c_infer = bo[j].theta + ctx->work.reward_cost_const + upd[k];
      const double objective = c_train < c_infer ? c_infer : c_train;  // std::max
      const long long mask = m0 + i;
      if (!have || objective < best) {
        have = true;
        best = objective;
        best_mask = mask;
      }
      if (c_infer >= c_train && (!have_c || objective < best_c)) {
        have_c = true;
        best_c = objective;
        best_mask_c = mask;
      }
    }
    out->partitions += q;
  }
  if (std::getenv("GPLAN_PROFILE"))
    std::fprintf(stderr, "exhaustive: train %.3f s, candidate counts %.3f s, configs %.3f s, brute MILP %.3f s, "
                 "weight sync %.3f s\n", ph[0], ph[1], ph[2], ph[3], ph[4]);
  out->feasible = have_c || have;
  out->objective = have_c ? best_c : best;
  const long long m = have_c ? best_mask_c : best_mask;
  if (out->feasible)
    for (int d = 0; d < N; ++d)
      if ((m >> d) & 1) train_ids[out->n_train++] = d;
  return GP_OK;
}

}  // namespace gp

extern "C" {

int gp_train_candidates_search(gp_ctx* ctx, const int32_t* ids, int32_t n, int32_t window,
                               gp_train_result* out, int32_t* stage_devices) {
  if (!ctx) return gp::set_error(GP_INVALID, "null context");
  if (!out || (n > 0 && (!ids || !stage_devices))) return gp::set_error(GP_INVALID, "null argument");
  cudaSetDevice(ctx->device);
  return gp::train_candidates_search(ctx, ids, n, window, out, stage_devices);
}

int gp_exhaustive_optimum(gp_ctx* ctx, int32_t window, gp_exhaustive_result* out, int32_t* train_ids) {
  if (!ctx) return gp::set_error(GP_INVALID, "null context");
  if (!out || !train_ids) return gp::set_error(GP_INVALID, "null argument");
  cudaSetDevice(ctx->device);
  return gp::exhaustive_optimum(ctx, window, out, train_ids);
}

}  // extern "C"
