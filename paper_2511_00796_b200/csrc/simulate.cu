// simulate.cu — the plan simulator: the event-level simulation of the
// asynchronous RL loop under a scheduled plan (src/simulator.cpp:70-403). The simulation is
// a serial discrete-event loop, so the GPU runs it replica-parallel: one thread per
// (plan, seed), each with its own replica table, FIFO rollout queue and event heap in a
// global-memory scratch slice. Every arithmetic step follows the reference in order
// (sequential token sums, the staleness gate, pause shifts), and the event order is the
// reference's (time, kind, sequence) order, so the reports are bit-identical.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <vector>

#include "gp_internal.h"

namespace gp {

namespace {

constexpr long long kEtaUnbounded = 1000000;  // src/simulator.cpp:29

struct SimReplica {
  double throughput, stall_start, batch_start, batch_end;
  long long version, batch_version, batch_reserved, epoch;
  unsigned long long rng;  // SplitMix64 state (inc/common.hpp:71-90)
  int capacity, batch_size;
  int generating, stalled;
};

struct SimQueued {
  long long version;
  long long output_len;
};

struct SimEvent {  // Pending (src/simulator.cpp:33-45): ordered by (time, kind, seq)
  double time;
  long long seq;
  long long epoch;
  int kind;  // 0 batch_done, 1 train_done, 2 sync_done
  int replica;
};

struct SimShared {  // per simulation set (identical for every seed)
  int n_rep, max_cap, n_buckets, batch_rollouts, prompt_len, steps, sync_every, window;
  long long eta, queue_cap, heap_cap;
  double train_time, sync_time, reward_time, per_hour;
};

__device__ __forceinline__ bool ev_less(const SimEvent& a, const SimEvent& b) {
  if (a.time != b.time) return a.time < b.time;
  if (a.kind != b.kind) return a.kind < b.kind;
  return a.seq < b.seq;
}

__device__ __forceinline__ unsigned long long sm64_next(unsigned long long& s) {
  unsigned long long z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double sm64_double(unsigned long long& s) {
  return static_cast<double>(sm64_next(s) >> 11) * 0x1.0p-53;
}

struct SimState {
  const SimShared& sh;
  const int* blen;
  const double* bcdf;
  SimReplica* rep;
  int* lens;  // [n_rep][max_cap] lengths of the current (or candidate) batch
  SimQueued* q;
  long long q_head = 0, q_size = 0;
  SimEvent* heap;
  long long heap_n = 0, seq = 0;
  long long trainer_version = 0;
  int steps_started = 0, steps_done = 0;
  bool training = false, syncing = false;
  double trainer_free_since = 0, train_step_start = 0;
  long long produced = 0, started = 0, consumed = 0, max_staleness = 0, tokens_consumed = 0;
  double stall_total = 0, wait_total = 0, roll_busy = 0, train_busy = 0, sync_total = 0, reward_total = 0;
  double* step_end;  // step_end_times
  int n_step_end = 0;
  int err = 0;

  __device__ SimState(const SimShared& s, const int* bl, const double* bc) : sh(s), blen(bl), bcdf(bc) {}

  __device__ int sample(double u) const {  // LengthDistribution::sample (src/workload.cpp:51-56)
    for (int i = 0; i < sh.n_buckets; ++i)
      if (u < bcdf[i]) return blen[i];
    return blen[sh.n_buckets - 1];
  }

  __device__ void push(double t, int kind, int replica, long long epoch) {
    if (heap_n >= sh.heap_cap) {
      err = GP_CAPACITY;
      return;
    }
    SimEvent e{t, seq++, epoch, kind, replica};
    long long i = heap_n++;
    while (i > 0) {
      const long long p = (i - 1) / 2;
      if (!ev_less(e, heap[p])) break;
      heap[i] = heap[p];
      i = p;
    }
    heap[i] = e;
  }

  __device__ SimEvent pop() {
    const SimEvent top = heap[0];
    const SimEvent last = heap[--heap_n];
    long long i = 0;
    while (true) {
      long long c = 2 * i + 1;
      if (c >= heap_n) break;
      if (c + 1 < heap_n && ev_less(heap[c + 1], heap[c])) ++c;
      if (!ev_less(heap[c], last)) break;
      heap[i] = heap[c];
      i = c;
    }
    if (heap_n > 0) heap[i] = last;
    return top;
  }

  __device__ long long rank_budget(long long version) const {
    return (long long)sh.batch_rollouts * sh.sync_every * (version + sh.eta + 1);
  }

  // gated_batch_size (src/simulator.cpp:121-150)
  __device__ int gated_batch_size(int idx, double now, int want) const {
    const SimReplica& r = rep[idx];
    if (sh.eta >= kEtaUnbounded) return want;
    const int* L = lens + (size_t)idx * sh.max_cap;
    int b = want;
    for (int guard = 0; guard <= sh.n_rep + 2 && b > 0; ++guard) {
      double tokens = 0;
      for (int i = 0; i < b; ++i) tokens += L[i];
      const double our_end = now + tokens / r.throughput;
      long long ahead = consumed + q_size;
      long long leapfrog = LLONG_MAX;
      for (int o = 0; o < sh.n_rep; ++o) {
        const SimReplica& other = rep[o];
        if (!other.generating) continue;
        if (other.batch_end >= our_end) leapfrog = min(leapfrog, rank_budget(other.batch_version) - other.batch_reserved);
        if (other.batch_end <= our_end) ahead += other.batch_size;
      }
      const long long own = rank_budget(r.version) - ahead;
      const long long cap = min(own, leapfrog);
      if (b <= cap) return b;
      b = (int)max(cap, 0LL);
    }
    return b;
  }

  // try_start_replica (src/simulator.cpp:152-204)
  __device__ void try_start_replica(int idx, double now) {
    SimReplica& r = rep[idx];
    if (r.generating || syncing) return;
    const int want = r.capacity;
    int* L = lens + (size_t)idx * sh.max_cap;
    for (int i = 0; i < want; ++i) L[i] = sample(sm64_double(r.rng));
    const int batch = gated_batch_size(idx, now, want);
    if (batch <= 0) {
      if (!r.stalled) {
        r.stalled = 1;
        r.stall_start = now;
      }
      return;
    }
    if (r.stalled) {
      r.stalled = 0;
      stall_total += now - r.stall_start;
    }
    double tokens = 0;
    for (int i = 0; i < batch; ++i) tokens += L[i];
    const double our_end = now + tokens / r.throughput;
    long long ahead = consumed + q_size;
    for (int o = 0; o < sh.n_rep; ++o) {
      SimReplica& other = rep[o];
      if (!other.generating) continue;
      if (other.batch_end >= our_end) other.batch_reserved += batch;
      if (other.batch_end <= our_end) ahead += other.batch_size;
    }
    r.generating = 1;
    r.batch_start = now;
    r.batch_version = r.version;
    r.batch_size = batch;
    r.batch_end = our_end;
    r.batch_reserved = ahead + batch;
    started += batch;
    push(r.batch_end, 0, idx, r.epoch);
  }

  // on_batch_done (src/simulator.cpp:206-219)
  __device__ void on_batch_done(int idx, double now) {
    SimReplica& r = rep[idx];
    r.generating = 0;
    produced += r.batch_size;
    roll_busy += now - r.batch_start;
    const int* L = lens + (size_t)idx * sh.max_cap;
    for (int i = 0; i < r.batch_size; ++i) {
      if (q_size >= sh.queue_cap) {
        err = GP_CAPACITY;
        return;
      }
      q[(q_head + q_size) % sh.queue_cap] = SimQueued{r.batch_version, (long long)L[i]};
      ++q_size;
    }
    try_start_training(now);
    try_start_replica(idx, now);
  }

  // try_start_training (src/simulator.cpp:221-244)
  __device__ void try_start_training(double now) {
    if (training || syncing) return;
    if (steps_started >= sh.steps) return;
    if (q_size < sh.batch_rollouts) return;
    for (int i = 0; i < sh.batch_rollouts; ++i) {
      const SimQueued ro = q[q_head];
      q_head = (q_head + 1) % sh.queue_cap;
      --q_size;
      const long long staleness = trainer_version - ro.version;
      max_staleness = max(max_staleness, staleness);
      tokens_consumed += sh.prompt_len + ro.output_len;
      consumed++;
    }
    wait_total += now - trainer_free_since;
    training = true;
    steps_started++;
    reward_total += sh.reward_time;
    roll_busy += sh.reward_time;
    train_step_start = now + sh.reward_time;
    push(train_step_start + sh.train_time, 1, -1, 0);
  }

  // on_train_done (src/simulator.cpp:246-272)
  __device__ void on_train_done(double now) {
    training = false;
    steps_done++;
    train_busy += sh.train_time;
    if (steps_done % sh.sync_every == 0) {
      syncing = true;
      sync_total += sh.sync_time;
      for (int i = 0; i < sh.n_rep; ++i) {
        SimReplica& r = rep[i];
        if (r.generating) {
          r.epoch++;
          r.batch_end += sh.sync_time;
          push(r.batch_end, 0, i, r.epoch);
        }
      }
      push(now + sh.sync_time, 2, -1, 0);
    } else {
      trainer_free_since = now;
      step_end[n_step_end++] = now;
      try_start_training(now);
    }
  }

  // on_sync_done (src/simulator.cpp:274-284)
  __device__ void on_sync_done(double now) {
    syncing = false;
    trainer_version++;
    for (int i = 0; i < sh.n_rep; ++i) rep[i].version = trainer_version;
    trainer_free_since = now;
    step_end[n_step_end++] = now;
    try_start_training(now);
    for (int i = 0; i < sh.n_rep; ++i)
      if (!rep[i].generating) try_start_replica(i, now);
  }
};

__global__ void k8_simulate(int n_seeds, const unsigned long long* __restrict__ seeds, SimShared sh,
                            const double* __restrict__ rep_tp, const int* __restrict__ rep_cap,
                            const int* __restrict__ blen, const double* __restrict__ bcdf, char* __restrict__ scratch,
                            size_t per_sim, gp_sim_report* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_seeds) return;
  char* base = scratch + per_sim * t;
  auto carve = [&](size_t bytes) {
    char* p = base;
    base += (bytes + 15) & ~size_t(15);
    return p;
  };
  SimState S(sh, blen, bcdf);
  S.rep = reinterpret_cast<SimReplica*>(carve(sizeof(SimReplica) * sh.n_rep));
  S.lens = reinterpret_cast<int*>(carve(sizeof(int) * (size_t)sh.n_rep * sh.max_cap));
  S.q = reinterpret_cast<SimQueued*>(carve(sizeof(SimQueued) * sh.queue_cap));
  S.heap = reinterpret_cast<SimEvent*>(carve(sizeof(SimEvent) * sh.heap_cap));
  S.step_end = reinterpret_cast<double*>(carve(sizeof(double) * (sh.steps + 1)));
  const unsigned long long seed = seeds[t];
  for (int i = 0; i < sh.n_rep; ++i) {  // src/simulator.cpp:297-318
    SimReplica& r = S.rep[i];
    r = SimReplica{};
    r.throughput = rep_tp[i];
    r.capacity = rep_cap[i];
    r.rng = seed ^ (0x9e3779b97f4a7c15ull * (static_cast<unsigned long long>(i) + 1));
  }
  for (int i = 0; i < sh.n_rep && !S.err; ++i) S.try_start_replica(i, 0.0);
  double now = 0;
  while (!S.err && (S.steps_done < sh.steps || S.syncing)) {
    if (S.heap_n == 0) {  // deadlock (src/simulator.cpp:326-328)
      S.err = GP_INVALID;
      break;
    }
    const SimEvent ev = S.pop();
    now = ev.time;
    if (ev.kind == 0) {
      SimReplica& r = S.rep[ev.replica];
      if (!r.generating || ev.epoch != r.epoch) continue;  // superseded by a pause
      S.on_batch_done(ev.replica, now);
    } else if (ev.kind == 1) {
      S.on_train_done(now);
    } else {
      S.on_sync_done(now);
    }
  }
  gp_sim_report o;
  memset(&o, 0, sizeof o);
  o.pad = S.err;
  if (!S.err) {  // src/simulator.cpp:343-366
    o.steps_completed = S.steps_done;
    o.total_time = now;
    o.max_staleness_observed = S.max_staleness;
    o.rollouts_produced = S.produced;
    o.rollouts_consumed = S.consumed;
    o.rollouts_pending = S.produced - S.consumed;
    o.rollouts_in_flight = S.started - S.produced;
    o.tokens_consumed = S.tokens_consumed;
    o.avg_step_time = now / sh.steps;
    const int warmup = min(sh.window, sh.steps - 1);
    if (warmup >= 1 && sh.steps > warmup) {
      const double warm_end = S.step_end[warmup - 1];
      o.avg_step_time_steady = (now - warm_end) / (sh.steps - warmup);
    } else {
      o.avg_step_time_steady = o.avg_step_time;
    }
    o.throughput_tokens_per_s = now > 0 ? static_cast<double>(S.tokens_consumed) / now : 0.0;
    o.rollout_stall_time = S.stall_total;
    o.trainer_wait_time = S.wait_total;
    o.rollout_busy_time = S.roll_busy;
    o.train_busy_time = S.train_busy;
    o.sync_time_total = S.sync_total;
    o.reward_time_total = S.reward_total;
    // dollar cost at simulated throughput (src/simulator.cpp:392-399)
    o.dollar_cost_per_token = o.throughput_tokens_per_s > 0 ? sh.per_hour / 3600.0 / o.throughput_tokens_per_s
                                                            : __longlong_as_double(0x7ff8000000000000LL);
  }
  out[t] = o;
}

// replica_concurrency (src/cost_model.cpp:128-148) of each entry config, as in K3.
__global__ void k8_concurrency(int n, const gp_config* __restrict__ cfg, Scalars sc, const double* __restrict__ tcap,
                               int T, int* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const gp_config c = cfg[i];
  int t = -1;
  for (int u = 0; u < T; ++u)
    if (c.type_counts[u] > 0) {
      t = u;
      break;
    }
  if (t < 0) {
    out[i] = 0;
    return;
  }
  int best = sc.max_conc;
  const int S = c.n_stages;
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
      const double q = free_b / kv;  // static_cast<int> as x86 cvttsd2si (INT_MIN out of range)
      const int v = (q >= 2147483648.0 || q < -2147483648.0 || q != q) ? INT_MIN : (int)q;
      best = v < best ? v : best;
    }
  }
  out[i] = best > 0 ? best : 0;
}

__global__ void k8_per_hour(const double* __restrict__ price, const int* __restrict__ ids, int n, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0;
  for (int i = 0; i < n; ++i) s += price[ids[i]];  // train set, then the bound rollout devices
  *out = s;
}

}  // namespace

int simulate(gp_ctx* ctx, const gp_sim_plan* p, int steps, int sync_every, const uint64_t* seeds, int n_seeds,
             gp_sim_report* out, int32_t* used_devices, int32_t* n_used) {
  if (steps < 1) return set_error(GP_INVALID, "simulation needs at least one step");
  if (n_seeds <= 0) return GP_OK;
  if (sync_every < 1) sync_every = 1;
  if (p->n_buckets < 1) return set_error(GP_INVALID, "length distribution must have at least one bucket");
  // LengthDistribution (src/workload.cpp:22-41): sorted (length, probability) pairs, cumulative
  std::vector<std::pair<int, double>> hist;
  for (int i = 0; i < p->n_buckets; ++i) hist.push_back({p->bucket_len[i], p->bucket_prob[i]});
  std::sort(hist.begin(), hist.end());
  std::vector<int> blen;
  std::vector<double> bcdf;
  double cum = 0;
  for (auto& h : hist) {
    cum += h.second;
    blen.push_back(h.first);
    bcdf.push_back(cum);
  }
  bcdf.back() = 1.0;
  // replicas and the concrete rollout devices bound to them (src/simulator.cpp:297-318)
  for (int i = 0; i < p->n_rollout; ++i)
    if (p->rollout_ids[i] < 0 || p->rollout_ids[i] >= ctx->N) return set_error(GP_INVALID, "unknown device id");
  for (int i = 0; i < p->n_train; ++i)
    if (p->train_ids[i] < 0 || p->train_ids[i] >= ctx->N) return set_error(GP_INVALID, "unknown device id");
  std::vector<std::vector<int>> free_by_type(ctx->T);
  for (int i = 0; i < p->n_rollout; ++i) free_by_type[ctx->h_type[p->rollout_ids[i]]].push_back(p->rollout_ids[i]);
  std::vector<size_t> taken(ctx->T, 0);
  std::vector<int> used, rep_entry;
  for (int e = 0; e < p->n_entries; ++e) {
    const gp_config& c = p->configs[e];
    int type = -1, per = 0;
    for (int u = 0; u < ctx->T; ++u) {
      if (c.type_counts[u] > 0 && type < 0) type = u;
      per += c.type_counts[u];
    }
    for (int k = 0; k < p->replicas[e]; ++k) {
      for (int d = 0; d < per; ++d) {
        if (type < 0 || taken[type] >= free_by_type[type].size())
          return set_error(GP_INVALID, "rollout plan needs more devices than the partition holds");
        used.push_back(free_by_type[type][taken[type]++]);
      }
      rep_entry.push_back(e);
    }
  }
  if (rep_entry.empty()) return set_error(GP_INVALID, "plan has no rollout replicas to simulate");
  if (used_devices) std::memcpy(used_devices, used.data(), sizeof(int32_t) * used.size());
  if (n_used) *n_used = (int32_t)used.size();
  const int n_rep = (int)rep_entry.size();
  // device inputs: configs, buckets, replica throughputs, price ids
  std::vector<int> price_ids(p->train_ids, p->train_ids + p->n_train);
  price_ids.insert(price_ids.end(), used.begin(), used.end());
  std::vector<double> rep_tp(n_rep);
  for (int i = 0; i < n_rep; ++i) rep_tp[i] = p->configs[rep_entry[i]].throughput;
  SimShared sh{};
  sh.n_rep = n_rep;
  sh.max_cap = std::max(1, ctx->sc.max_conc);
  sh.n_buckets = (int)blen.size();
  sh.batch_rollouts = ctx->work.batch_rollouts;
  sh.prompt_len = ctx->work.prompt_len;
  sh.steps = steps;
  sh.sync_every = sync_every;
  sh.window = p->window;
  sh.eta = std::min<long long>(p->staleness, kEtaUnbounded);  // the plan's staleness (src/cli.cpp:193)
  sh.train_time = p->c_train / p->window;
  sh.sync_time = p->c_update / p->window;
  sh.reward_time = p->c_reward / p->window;
  // queue: at most every rollout begun (steps consumed + one capacity-sized batch per replica
  // per version the gate admits); heap: every live batch plus one stale event per pause
  const long long begun_bound =
      (long long)sh.batch_rollouts * sync_every * (steps + std::min<long long>(sh.eta, steps) + 2) +
      (long long)n_rep * sh.max_cap * 4;
  sh.queue_cap = sh.eta >= kEtaUnbounded ? (long long)sh.batch_rollouts * (steps + 2) + (long long)n_rep * sh.max_cap * 64
                                         : begun_bound;
  sh.heap_cap = (long long)n_rep * (steps / sync_every + 2) + 8;
  const size_t per_sim = ((sizeof(SimReplica) * n_rep + 15) & ~15) + ((sizeof(int) * n_rep * sh.max_cap + 15) & ~15) +
                         ((sizeof(SimQueued) * sh.queue_cap + 15) & ~15) + ((sizeof(SimEvent) * sh.heap_cap + 15) & ~15) +
                         ((sizeof(double) * (steps + 1) + 15) & ~15);
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += ((b + 255) & ~size_t(255)) + 256; };
  add(sizeof(gp_config) * p->n_entries);
  add(sizeof(int) * p->n_entries);
  add(sizeof(int) * blen.size());
  add(sizeof(double) * bcdf.size());
  add(sizeof(double) * n_rep);
  add(sizeof(int) * n_rep);
  add(sizeof(int) * (price_ids.size() + 1));
  add(sizeof(double) * ctx->N);
  add(sizeof(double));
  add(sizeof(unsigned long long) * n_seeds);
  add(sizeof(gp_sim_report) * n_seeds);
  add(per_sim * n_seeds);
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  char* base = static_cast<char*>(ctx_scratch(ctx, bytes, kArenaMisc));
  if (!base) return GP_CUDA_ERROR;
  char* q = base;
  auto carve = [&](size_t b) {
    q = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(q) + 255) & ~uintptr_t(255));
    char* r = q;
    q += b;
    return r;
  };
  gp_config* d_cfg = reinterpret_cast<gp_config*>(carve(sizeof(gp_config) * p->n_entries));
  int* d_conc = reinterpret_cast<int*>(carve(sizeof(int) * p->n_entries));
  int* d_blen = reinterpret_cast<int*>(carve(sizeof(int) * blen.size()));
  double* d_bcdf = reinterpret_cast<double*>(carve(sizeof(double) * bcdf.size()));
  double* d_reptp = reinterpret_cast<double*>(carve(sizeof(double) * n_rep));
  int* d_repcap = reinterpret_cast<int*>(carve(sizeof(int) * n_rep));
  int* d_pids = reinterpret_cast<int*>(carve(sizeof(int) * (price_ids.size() + 1)));
  double* d_price = reinterpret_cast<double*>(carve(sizeof(double) * ctx->N));
  double* d_perhour = reinterpret_cast<double*>(carve(sizeof(double)));
  unsigned long long* d_seeds = reinterpret_cast<unsigned long long*>(carve(sizeof(unsigned long long) * n_seeds));
  gp_sim_report* d_out = reinterpret_cast<gp_sim_report*>(carve(sizeof(gp_sim_report) * n_seeds));
  char* d_scratch = carve(per_sim * n_seeds);
  auto up = [&](void* d, const void* h, size_t b) -> int {
    if (b) GP_CUDA(cudaMemcpyAsync(d, h, b, cudaMemcpyHostToDevice, ctx->stream));
    ctx->h2d_bytes += (long long)b;
    return GP_OK;
  };
  int rc = up(d_cfg, p->configs, sizeof(gp_config) * p->n_entries);
  if (!rc) rc = up(d_blen, blen.data(), sizeof(int) * blen.size());
  if (!rc) rc = up(d_bcdf, bcdf.data(), sizeof(double) * bcdf.size());
  if (!rc) rc = up(d_reptp, rep_tp.data(), sizeof(double) * n_rep);
  if (!rc) rc = up(d_pids, price_ids.data(), sizeof(int) * price_ids.size());
  if (!rc) rc = up(d_price, p->device_price, sizeof(double) * ctx->N);
  if (!rc) rc = up(d_seeds, seeds, sizeof(unsigned long long) * n_seeds);
  if (rc) return rc;
  k8_concurrency<<<(p->n_entries + 127) / 128 + 1, 128, 0, ctx->stream>>>(p->n_entries, d_cfg, ctx->sc, ctx->d_tcap,
                                                                        ctx->T, d_conc);
  k8_per_hour<<<1, 32, 0, ctx->stream>>>(d_price, d_pids, (int)price_ids.size(), d_perhour);
  ctx->launches += 2;
  std::vector<int> conc(p->n_entries);
  double per_hour = 0;
  GP_CUDA(cudaMemcpyAsync(conc.data(), d_conc, sizeof(int) * p->n_entries, cudaMemcpyDeviceToHost, ctx->stream));
  GP_CUDA(cudaMemcpyAsync(&per_hour, d_perhour, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  std::vector<int> rep_cap(n_rep);  // std::max(1, concurrency) <= max(1, max_concurrency) = sh.max_cap
  for (int i = 0; i < n_rep; ++i) rep_cap[i] = std::max(1, conc[rep_entry[i]]);
  sh.per_hour = per_hour;
  rc = up(d_repcap, rep_cap.data(), sizeof(int) * n_rep);
  if (rc) return rc;
  k8_simulate<<<(n_seeds + 63) / 64, 64, 0, ctx->stream>>>(n_seeds, d_seeds, sh, d_reptp, d_repcap, d_blen, d_bcdf,
                                                          d_scratch, per_sim, d_out);
  ctx->launches++;
  GP_CUDA(cudaGetLastError());
  GP_CUDA(cudaMemcpyAsync(out, d_out, sizeof(gp_sim_report) * n_seeds, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->d2h_bytes += (long long)(sizeof(gp_sim_report) * n_seeds);
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < n_seeds; ++i) {
    const int err = out[i].pad;
    out[i].pad = 0;
    if (err == GP_INVALID) return set_error(GP_INVALID, "simulation deadlocked; plan and workload are inconsistent");
    if (err) return set_error(GP_CAPACITY, "simulation queue or event heap exceeded its bound");
  }
  return GP_OK;
}

}  // namespace gp

extern "C" int gp_simulate(gp_ctx* ctx, const gp_sim_plan* plan, int32_t steps, int32_t sync_every,
                           const uint64_t* seeds, int32_t n_seeds, gp_sim_report* out, int32_t* used_devices,
                           int32_t* n_used) {
  if (!ctx) return gp::set_error(GP_INVALID, "null context");
  if (!plan || (n_seeds > 0 && (!seeds || !out))) return gp::set_error(GP_INVALID, "null argument");
  cudaSetDevice(ctx->device);
  return gp::simulate(ctx, plan, steps, sync_every, seeds, n_seeds, out, used_devices, n_used);
}
