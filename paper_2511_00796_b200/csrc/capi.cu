// capi.cu — extern "C" entry points of libgplan.so (include/gplan.h) and the
// engine context: validation, device upload, scratch management, error state.
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "gp_internal.h"

namespace gp {

int train_space(gp_ctx* ctx, const int32_t* ids, int n, const gp_train_opts* o, int64_t* layouts);
int train_search(gp_ctx* ctx, const int32_t* ids, int n, int window, const gp_train_opts* o,
                 long long lo, long long hi, gp_train_result* out, int32_t* stage_devices, int mode = 0);
int train_prepare(gp_ctx* ctx, const int32_t* ids, int n, const gp_train_opts* o, int mode = 0);
int train_launch(gp_ctx* ctx, int window, long long lo, long long hi);
int train_collect(gp_ctx* ctx, gp_train_result* out, int32_t* stage_devices);
int train_layout_costs(gp_ctx* ctx, const int32_t* ids, int n, const gp_train_opts* o, long long lo,
                       long long hi, int path, double* out, int* fast_used, int* inner);
int train_shard_bounds(gp_ctx* ctx, const int32_t* ids, int n, const gp_train_opts* o, int n_shards,
                       int64_t* bounds);
int train_batch(gp_ctx* ctx, int n_sets, const int32_t* const* ids, const int32_t* ns, int window,
                const gp_train_opts* o, gp_train_result* outs, int32_t* const* stage_devices, int mode);
void train_state_free(gp_ctx* ctx);
void train_last_nm(gp_ctx* ctx, long long nm[4]);
void train_nm_merge(long long a[4], const long long b[4]);
void train_memo_free(gp_ctx* ctx);
std::string train_memo_key(const int32_t* ids, int n, const gp_train_opts* o, int mode = 0);
bool train_memo_get(gp_ctx* ctx, const std::string& key, int window, gp_train_result* out,
                    int32_t* stage_devices);
void train_memo_put_last(gp_ctx* ctx, const std::string& key, const gp_train_result& r, const long long nm[4]);
void milp_cache_free(gp_ctx* ctx);
void part_cache_free(gp_ctx* ctx);
int rollout_configs(gp_ctx* ctx, const int32_t* ids, int n, const gp_rollout_opts* o, gp_config* out,
                    int cap, int* n_out);
int rollout_capacities(gp_ctx* ctx, const int32_t* ids, int n, int32_t* caps);
int solve_milp(gp_ctx* ctx, const gp_config* cfg, int nc, const int32_t* caps, int dims, double B,
               double len, gp_rollout_result* out, gp_rollout_entry* entries);
int milp_batch(gp_ctx* ctx, int q, const gp_config* const* cfgs, const int* ncs, const int32_t* const* caps,
               int dims, const double* Bs, double len, gp_rollout_result* outs, gp_rollout_entry* const* entries,
               int* rcs);
int weight_sync(gp_ctx* ctx, const int32_t* train, int nt, const int32_t* roll, int nr,
                const int32_t* etype, const int32_t* erep, int ne, int window, double* out);
int partition_candidates(gp_ctx* ctx, const gp_gamma* g, const gp_part_opts* o, int k, gp_partition* out,
                         int32_t* train_ids, int32_t* n_out);
int partition_objective(gp_ctx* ctx, const int32_t* train, int nt, double* obj, double* frac);
int compute_fraction(gp_ctx* ctx, const int32_t* train, int nt, double* frac);
int schedule(gp_ctx* ctx, const gp_sched_opts* o, gp_schedule_result* res, int32_t* train_ids,
             int32_t* rollout_ids, int32_t* stage_devices, gp_config* entry_configs, gp_rollout_entry* entries,
             int32_t entry_cap, double* trace);

static thread_local std::string g_error;

int set_error(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return set_error(GP_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

void* ctx_scratch(gp_ctx* ctx, size_t bytes, int arena) {
  void*& buf = ctx->scratch_arena[arena];
  size_t& have = ctx->scratch_arena_bytes[arena];
  if (bytes > have) {
    // stream-ordered (the device's pool): a grown arena does not synchronise the whole device,
    // which other host threads (peer / auxiliary contexts on the same GPU) may be using. Every
    // API call ends with ctx->stream synchronised after its lane streams, so the old buffer
    // is idle when it is released.
    if (buf) cudaFreeAsync(buf, ctx->stream);
    buf = nullptr;
    // 1.5x headroom with a 4 MiB floor: the scheduler's batches vary in size and a
    // cudaMalloc/cudaFree pair costs more than the kernels of a small batch
    size_t want = std::max(bytes + bytes / 2, (size_t)4 << 20);
    cudaError_t e = cudaMallocAsync(&buf, want, ctx->stream);
    if (e != cudaSuccess) {
      have = 0;
      cuda_fail(e, "cudaMalloc(scratch)");
      return nullptr;
    }
    have = want;
  }
  return buf;
}

void* ctx_pinned(gp_ctx* ctx, size_t bytes) {
  if (bytes > ctx->h_pinned_bytes) {
    if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
    ctx->h_pinned = nullptr;
    size_t want = std::max(bytes + bytes / 2 + 4096, (size_t)4 << 20);
    cudaError_t e = cudaMallocHost(&ctx->h_pinned, want);
    if (e != cudaSuccess) {
      ctx->h_pinned_bytes = 0;
      cuda_fail(e, "cudaMallocHost(staging)");
      return nullptr;
    }
    ctx->h_pinned_bytes = want;
  }
  return ctx->h_pinned;
}

__global__ void k_probe(int* flag) { *flag = 0x5eed; }

// GP_SEGV_TRACE=1: print a native backtrace on SIGSEGV (debug aid on GPU boxes without gdb).
static void segv_handler(int sig) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  const char msg[] = "libgplan: fatal signal, native backtrace:\n";
  (void)!write(2, msg, sizeof msg - 1);
  backtrace_symbols_fd(frames, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}

// Every device of a type carries the same capabilities in the reference loader
// (src/cluster.cpp:127-137); the engine's rollout side relies on it.
static int validate(const gp_cluster* c, const gp_workload* w, const gp_calib* k) {
  if (!c || !w || !k) return set_error(GP_INVALID, "null input");
  if (c->n_devices < 1) return set_error(GP_INVALID, "cluster has no devices");
  if (c->n_types < 1 || c->n_types > GP_MAX_TYPES)
    return set_error(GP_INVALID, "n_types must lie in [1, GP_MAX_TYPES]");
  if (c->n_machines < 1) return set_error(GP_INVALID, "cluster has no machines");
  for (int d = 0; d < c->n_devices; ++d) {
    if (c->device_type[d] < 0 || c->device_type[d] >= c->n_types)
      return set_error(GP_INVALID, "device " + std::to_string(d) + " has an unknown gpu_type");
    if (c->device_machine[d] < 0 || c->device_machine[d] >= c->n_machines)
      return set_error(GP_INVALID, "device " + std::to_string(d) + " has an unknown machine");
  }
  // WorkloadSpec::validate (src/workload.cpp:58-69)
  if (!(w->model_params_b > 0)) return set_error(GP_INVALID, "model.params_billion must be > 0");
  if (w->num_layers < 1) return set_error(GP_INVALID, "model.num_layers must be >= 1");
  if (w->hidden_dim < 1) return set_error(GP_INVALID, "model.hidden_dim must be >= 1");
  if (w->batch_rollouts < 1) return set_error(GP_INVALID, "batch_rollouts must be >= 1");
  if (w->prompt_len < 0) return set_error(GP_INVALID, "prompt_len must be >= 0");
  if (!(w->bytes_per_param_train > 0)) return set_error(GP_INVALID, "bytes_per_param_train must be > 0");
  if (!(w->bytes_per_param_infer > 0)) return set_error(GP_INVALID, "bytes_per_param_infer must be > 0");
  if (w->micro_batches < 1) return set_error(GP_INVALID, "micro_batches must be >= 1");
  return GP_OK;
}

// An auxiliary context on ctx's device for the driver's speculative partitions (schedule.cu),
// rebuilt from ctx's own copies of the inputs.
int ctx_make_aux(gp_ctx* ctx) {
  if (ctx->aux) return GP_OK;
  std::vector<double> links((size_t)ctx->N * ctx->N);
  GP_CUDA(cudaSetDevice(ctx->device));
  GP_CUDA(cudaMemcpy(links.data(), ctx->d_links, sizeof(double) * links.size(), cudaMemcpyDeviceToHost));
  gp_cluster c{ctx->N, ctx->T, ctx->M, ctx->h_type.data(), ctx->h_machine.data(), ctx->h_flops.data(),
               ctx->h_hbm_bw.data(), ctx->h_hbm_cap.data(), ctx->h_tflops.data(), ctx->h_thbm.data(),
               ctx->h_tcap.data(), links.data()};
  gp_calib k = ctx->calib;
  k.compute_eff = ctx->h_ceff.data();
  k.io_eff = ctx->h_ioeff.data();
  return gp_ctx_create(&c, &ctx->work, &k, ctx->device, &ctx->aux);
}
}  // namespace gp

using namespace gp;

extern "C" {

int gp_abi_version(void) { return GP_ABI_VERSION; }
const char* gp_last_error(void) { return g_error.c_str(); }

int gp_ctx_create(const gp_cluster* c, const gp_workload* w, const gp_calib* k, int device,
                  gp_ctx** out) {
  *out = nullptr;
  if (std::getenv("GP_SEGV_TRACE")) signal(SIGSEGV, segv_handler);
  int rc = validate(c, w, k);
  if (rc) return rc;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return set_error(GP_CUDA_ERROR, std::string("no CUDA device available (") +
                                        (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices") +
                                        "); the engine has no CPU fallback");
  if (device < 0 || device >= ndev) return set_error(GP_CUDA_ERROR, "CUDA ordinal out of range");
  GP_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  GP_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return set_error(GP_CUDA_ERROR, std::string("device ") + prop.name +
                                        " is not sm_100 (Blackwell); libgplan is built for sm_100a only");
  gp_ctx* ctx = new gp_ctx();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  const int N = c->n_devices, T = c->n_types;
  ctx->N = N;
  ctx->T = T;
  ctx->M = c->n_machines;
  ctx->h_type.assign(c->device_type, c->device_type + N);
  ctx->h_machine.assign(c->device_machine, c->device_machine + N);
  ctx->h_flops.assign(c->device_flops, c->device_flops + N);
  ctx->h_hbm_bw.assign(c->device_hbm_bw, c->device_hbm_bw + N);
  ctx->h_hbm_cap.assign(c->device_hbm_cap, c->device_hbm_cap + N);
  ctx->h_tflops.assign(c->type_flops, c->type_flops + T);
  ctx->h_thbm.assign(c->type_hbm_bw, c->type_hbm_bw + T);
  ctx->h_tcap.assign(c->type_hbm_cap, c->type_hbm_cap + T);
  ctx->h_ceff.assign(k->compute_eff, k->compute_eff + T);
  ctx->h_ioeff.assign(k->io_eff, k->io_eff + T);
  ctx->work = *w;
  ctx->calib = *k;
  ctx->calib.compute_eff = nullptr;
  ctx->calib.io_eff = nullptr;
  // derived scalars, same expressions as inc/workload.hpp:51-58
  Scalars& s = ctx->sc;
  s.P = w->model_params_b * 1e9;
  s.mtl = w->prompt_len + w->mean_len;
  s.tokens = w->batch_rollouts * s.mtl;
  s.tfpt_tokens = 6.0 * s.P * s.tokens;
  s.mbi = s.P * w->bytes_per_param_infer;
  s.ifpt = 2.0 * s.P;
  s.kvbpt = 4.0 * w->hidden_dim * w->num_layers;
  s.act_tok_h2 = s.tokens * w->hidden_dim * kActBytes;
  s.bpp_train = w->bytes_per_param_train;
  s.bpp_infer = w->bytes_per_param_infer;
  s.act_coeff = k->activation_coeff;
  s.tp_coeff = k->tp_allreduce_coeff;
  s.grad_bpp = k->grad_bytes_per_param;
  s.stage_pen = k->stage_latency_penalty;
  s.sync_latency = k->sync_latency_s;
  s.reward = w->reward_cost_const;
  s.L = w->num_layers;
  s.H = w->hidden_dim;
  s.mb = w->micro_batches;
  s.max_conc = k->max_concurrency;
  s.batch = w->batch_rollouts;
  s.mean_len = w->mean_len;

  auto fail = [&](int code) {
    gp_ctx_destroy(ctx);
    return code;
  };
#define UP(dst, src, count, T_)                                                           \
  do {                                                                                     \
    if (cudaMalloc(&dst, sizeof(T_) * (count)) != cudaSuccess)                             \
      return fail(set_error(GP_CUDA_ERROR, "cudaMalloc failed"));                          \
    if (cudaMemcpy(dst, src, sizeof(T_) * (count), cudaMemcpyHostToDevice) != cudaSuccess) \
      return fail(set_error(GP_CUDA_ERROR, "cudaMemcpy failed"));                          \
  } while (0)
  UP(ctx->d_type, c->device_type, N, int);
  UP(ctx->d_machine, c->device_machine, N, int);
  UP(ctx->d_flops, c->device_flops, N, double);
  UP(ctx->d_hbm_bw, c->device_hbm_bw, N, double);
  UP(ctx->d_hbm_cap, c->device_hbm_cap, N, double);
  UP(ctx->d_links, c->links, (size_t)N * N, double);
  UP(ctx->d_ceff, k->compute_eff, T, double);
  UP(ctx->d_ioeff, k->io_eff, T, double);
  UP(ctx->d_tflops, c->type_flops, T, double);
  UP(ctx->d_thbm, c->type_hbm_bw, T, double);
  UP(ctx->d_tcap, c->type_hbm_cap, T, double);
  {  // machine-structured links? (exact check over every ordered device pair)
    const int M = ctx->M;
    std::vector<double> ml((size_t)M * M, 0.0);
    std::vector<char> seen((size_t)M * M, 0);
    const char* dl = std::getenv("GPLAN_DEVICE_LINKS");  // force the device-level path (tests)
    bool ok = M > 0 && !(dl && dl[0] == '1');
    for (int a = 0; a < N && ok; ++a)
      for (int b = 0; b < N; ++b) {
        if (a == b) continue;
        const size_t slot = (size_t)c->device_machine[a] * M + c->device_machine[b];
        const double v = c->links[(size_t)a * N + b];
        if (!seen[slot]) {
          seen[slot] = 1;
          ml[slot] = v;
        } else if (std::memcmp(&ml[slot], &v, sizeof v) != 0) {
          ok = false;
          break;
        }
      }
    if (ok) UP(ctx->d_mlinks, ml.data(), (size_t)M * M, double);
  }
#undef UP
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(set_error(GP_CUDA_ERROR, "cudaStreamCreate failed"));
  {  // the scratch arenas and MILP tables are stream-ordered allocations: keep freed blocks
     // in the device pool instead of returning them at every synchronisation
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  // kernel-image probe: fails loudly if this build has no sm_100a code for the device
  int* flag = static_cast<int*>(ctx_scratch(ctx, 1 << 20));
  if (!flag) return fail(GP_CUDA_ERROR);
  k_probe<<<1, 1, 0, ctx->stream>>>(flag);
  int hflag = 0;
  cudaError_t pe = cudaGetLastError();
  if (pe == cudaSuccess) pe = cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
  if (pe == cudaSuccess) pe = cudaStreamSynchronize(ctx->stream);
  if (pe != cudaSuccess || hflag != 0x5eed)
    return fail(set_error(GP_CUDA_ERROR, std::string("kernel probe failed: ") + cudaGetErrorString(pe)));
  *out = ctx;
  return GP_OK;
}

void gp_ctx_destroy(gp_ctx* ctx) {
  if (!ctx) return;
  for (gp_ctx* peer : ctx->peers) gp_ctx_destroy(peer);
  ctx->peers.clear();
  gp_ctx_destroy(ctx->aux);
  ctx->aux = nullptr;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  void* ptrs[] = {ctx->d_type, ctx->d_machine, ctx->d_flops, ctx->d_hbm_bw, ctx->d_hbm_cap,
                  ctx->d_links, ctx->d_ceff, ctx->d_ioeff, ctx->d_tflops, ctx->d_thbm,
                  ctx->d_tcap,   ctx->d_mlinks, ctx->scratch_arena[0], ctx->scratch_arena[1],
                  ctx->scratch_arena[2], ctx->scratch_arena[3]};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  train_state_free(ctx);
  train_memo_free(ctx);
  if (ctx->d_slow) cudaFree(ctx->d_slow);
  for (int l = 0; l < gp_ctx::kTrainLanes; ++l) {
    if (ctx->d_slow_lane[l]) cudaFree(ctx->d_slow_lane[l]);
    if (ctx->lane[l]) cudaStreamDestroy(ctx->lane[l]);
  }
  for (auto& e : ctx->ev_lane)
    if (e) cudaEventDestroy(e);
  milp_cache_free(ctx);
  part_cache_free(ctx);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

long long gp_ctx_launches(gp_ctx* ctx) { return ctx ? ctx->launches : 0; }
void* gp_ctx_stream(gp_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int gp_train_space(gp_ctx* ctx, const int32_t* ids, int32_t n, const gp_train_opts* o,
                   int64_t* layouts) {
  if (!ctx) return set_error(GP_INVALID, "null context");
  return train_space(ctx, ids, n, o, layouts);
}

// In-call multi-GPU fan-out: a multi-device context splits the rank
// range of one search into contiguous shards, one per device; every device builds its
// tables and scans its shard on its own stream concurrently; the (cost, rank) winners
// are reduced lexicographically on the host (first rank among equal costs).
static int search_fanout(gp_ctx* ctx, const int32_t* ids, int32_t n, int32_t window,
                         const gp_train_opts* o, int64_t lo, int64_t hi, gp_train_result* out,
                         int32_t* stage_devices, long long nm[4]) {
  int64_t total = 0;
  int rc = train_space(ctx, ids, n, o, &total);
  if (rc) return rc;
  if (lo < 0) lo = 0;
  if (hi < 0 || hi > total) hi = total;
  if (lo > hi) lo = hi;
  const int P = 1 + (int)ctx->peers.size();
  if (ctx->peers.empty() || hi - lo < kFanoutMinLayouts) {
    cudaSetDevice(ctx->device);
    rc = train_search(ctx, ids, n, window, o, lo, hi, out, stage_devices);
    if (!rc) train_last_nm(ctx, nm);
    return rc;
  }
  std::vector<gp_ctx*> devs{ctx};
  devs.insert(devs.end(), ctx->peers.begin(), ctx->peers.end());
  std::vector<int64_t> bounds(P + 1);
  if (lo == 0 && hi == total) {  // whole space: shards that keep K1-fast's best scan order
    rc = train_shard_bounds(ctx, ids, n, o, P, bounds.data());
    if (rc) return rc;
  } else {
    for (int i = 0; i <= P; ++i) bounds[i] = lo + (hi - lo) * i / P;
  }
  int launched = 0;
  for (int i = 0; i < P && !rc; ++i) {  // enqueue everything first: shards run concurrently
    cudaSetDevice(devs[i]->device);
    rc = train_prepare(devs[i], ids, n, o);
    if (!rc) rc = train_launch(devs[i], window, bounds[i], bounds[i + 1]);
    if (!rc) ++launched;
  }
  if (rc) {  // drain the shards already running before reporting the error
    const std::string err = gp_last_error();
    for (int i = 0; i < launched; ++i) {
      cudaSetDevice(devs[i]->device);
      cudaStreamSynchronize(devs[i]->stream);
    }
    cudaSetDevice(ctx->device);
    return set_error(rc, err);
  }
  std::memset(out, 0, sizeof *out);
  out->layouts = hi - lo;
  nm[0] = 0x7ff0000000000000LL;
  nm[1] = nm[2] = nm[3] = LLONG_MAX;
  std::vector<int32_t> tmp(n > 0 ? n : 1);
  for (int i = 0; i < P; ++i) {
    cudaSetDevice(devs[i]->device);
    gp_train_result r;
    rc = train_collect(devs[i], &r, tmp.data());
    if (rc) return rc;
    long long nmi[4];
    train_last_nm(devs[i], nmi);
    train_nm_merge(nm, nmi);
    out->feasible += r.feasible;
    if (r.found && (!out->found || r.cost < out->cost || (r.cost == out->cost && r.rank < out->rank))) {
      const int64_t layouts = out->layouts, feasible = out->feasible;
      *out = r;
      out->layouts = layouts;
      out->feasible = feasible;
      if (stage_devices) std::memcpy(stage_devices, tmp.data(), sizeof(int32_t) * n);
    }
  }
  cudaSetDevice(ctx->device);
  return GP_OK;
}

int gp_constrained_search(gp_ctx* ctx, const int32_t* ids, int32_t n, int32_t window,
                          const gp_train_opts* o, gp_train_result* out, int32_t* stage_devices) {
  NvtxRange nvtx("gp_constrained_search");
  if (!ctx) return set_error(GP_INVALID, "null context");
  std::string key;
  if (ids && o && n > 0) {
    key = train_memo_key(ids, n, o);
    if (train_memo_get(ctx, key, window, out, stage_devices)) return GP_OK;
  }
  long long nm[4];
  const int rc = search_fanout(ctx, ids, n, window, o, 0, -1, out, stage_devices, nm);
  if (!rc && !key.empty()) train_memo_put_last(ctx, key, *out, nm);
  return rc;
}

int gp_constrained_search_range(gp_ctx* ctx, const int32_t* ids, int32_t n, int32_t window,
                                const gp_train_opts* o, int64_t lo, int64_t hi,
                                gp_train_result* out, int32_t* stage_devices) {
  NvtxRange nvtx("gp_constrained_search_range");
  if (!ctx) return set_error(GP_INVALID, "null context");
  long long nm[4];  // explicit ranges are never memoised: every call scans its range
  return search_fanout(ctx, ids, n, window, o, lo, hi, out, stage_devices, nm);
}


int gp_ctx_create_multi(const gp_cluster* c, const gp_workload* w, const gp_calib* k,
                        const int* devices, int n_devices, gp_ctx** out) {
  *out = nullptr;
  if (!devices || n_devices < 1) return set_error(GP_INVALID, "need at least one device");
  gp_ctx* primary = nullptr;
  int rc = gp_ctx_create(c, w, k, devices[0], &primary);
  if (rc) return rc;
  for (int i = 1; i < n_devices; ++i) {
    gp_ctx* peer = nullptr;
    rc = gp_ctx_create(c, w, k, devices[i], &peer);
    if (rc) {
      gp_ctx_destroy(primary);
      return rc;
    }
    primary->peers.push_back(peer);
  }
  if (n_devices > 1) {  // the scheduler's speculative-partition context (last device)
    rc = gp_ctx_create(c, w, k, devices[n_devices - 1], &primary->aux);
    if (rc) {
      gp_ctx_destroy(primary);
      return rc;
    }
  }
  cudaSetDevice(primary->device);
  *out = primary;
  return GP_OK;
}

int gp_train_prepare(gp_ctx* ctx, const int32_t* ids, int32_t n, const gp_train_opts* o) {
  NvtxRange nvtx("gp_train_prepare");
  if (!ctx) return set_error(GP_INVALID, "null context");
  cudaSetDevice(ctx->device);
  return train_prepare(ctx, ids, n, o);
}

int gp_constrained_search_batch(gp_ctx* ctx, int32_t n_sets, const int32_t* ids, const int32_t* off,
                                int32_t window, const gp_train_opts* o, gp_train_result* out,
                                int32_t* stage_devices) {
  NvtxRange nvtx("gp_constrained_search_batch");
  if (!ctx || !ids || !off || !out || n_sets < 0) return set_error(GP_INVALID, "null argument");
  const gp_train_opts def{4, 16};
  if (!o) o = &def;
  std::vector<const int32_t*> p(n_sets);
  std::vector<int32_t> ns(n_sets);
  std::vector<int32_t*> sd(n_sets);
  for (int i = 0; i < n_sets; ++i) {
    if (off[i + 1] < off[i]) return set_error(GP_INVALID, "set offsets must be non-decreasing");
    p[i] = ids + off[i];
    ns[i] = off[i + 1] - off[i];
    if (ns[i] <= 0) return set_error(GP_INVALID, "constrained_search requires a non-empty train set");
    sd[i] = stage_devices ? stage_devices + off[i] : nullptr;
  }
  cudaSetDevice(ctx->device);
  return train_batch(ctx, n_sets, p.data(), ns.data(), window, o, out, stage_devices ? sd.data() : nullptr, 0);
}

int gp_train_launch(gp_ctx* ctx, int32_t window, int64_t lo, int64_t hi) {
  NvtxRange nvtx("gp_train_launch");
  if (!ctx) return set_error(GP_INVALID, "null context");
  cudaSetDevice(ctx->device);
  return train_launch(ctx, window, lo, hi);
}

int gp_train_collect(gp_ctx* ctx, gp_train_result* out, int32_t* stage_devices) {
  NvtxRange nvtx("gp_train_collect");
  if (!ctx) return set_error(GP_INVALID, "null context");
  cudaSetDevice(ctx->device);
  return train_collect(ctx, out, stage_devices);
}

int gp_debug_layout_costs(gp_ctx* ctx, const int32_t* ids, int32_t n, const gp_train_opts* opts,
                          int64_t lo, int64_t hi, int32_t path, double* per_step, int32_t* fast_used) {
  if (!ctx || !per_step) return set_error(GP_INVALID, "null argument");
  cudaSetDevice(ctx->device);
  const gp_train_opts def{4, 16};
  int f = 0, inner = -1;
  const int rc = train_layout_costs(ctx, ids, n, opts ? opts : &def, lo, hi, path, per_step, &f, &inner);
  if (fast_used) *fast_used = f ? 1 + inner : 0;  // 1 + K1-fast's inner run, 0: generic K1
  return rc;
}

int gp_train_shard_bounds(gp_ctx* ctx, const int32_t* ids, int32_t n, const gp_train_opts* opts,
                          int32_t n_shards, int64_t* bounds) {
  if (!ctx || !bounds) return set_error(GP_INVALID, "null argument");
  const gp_train_opts def{4, 16};
  return train_shard_bounds(ctx, ids, n, opts ? opts : &def, n_shards, bounds);
}

int gp_enumerate_configs(gp_ctx* ctx, const int32_t* ids, int32_t n, const gp_rollout_opts* o,
                         gp_config* out, int32_t cap, int32_t* n_out) {
  NvtxRange nvtx("gp_enumerate_configs");
  if (!ctx) return set_error(GP_INVALID, "null context");
  cudaSetDevice(ctx->device);
  return rollout_configs(ctx, ids, n, o, out, cap, n_out);
}

int gp_rollout_capacities(gp_ctx* ctx, const int32_t* ids, int32_t n, int32_t* caps) {
  if (!ctx) return set_error(GP_INVALID, "null context");
  return rollout_capacities(ctx, ids, n, caps);
}

int gp_solve_milp(gp_ctx* ctx, const gp_config* configs, int32_t n_configs, const int32_t* caps,
                  int32_t dims, double total_rollouts, double mean_len, gp_rollout_result* out,
                  gp_rollout_entry* entries) {
  NvtxRange nvtx("gp_solve_milp");
  if (!ctx) return set_error(GP_INVALID, "null context");
  cudaSetDevice(ctx->device);
  return solve_milp(ctx, configs, n_configs, caps, dims, total_rollouts, mean_len, out, entries);
}

int gp_solve_milp_batch(gp_ctx* ctx, int32_t q, const gp_config* configs, const int32_t* cfg_off,
                        const int32_t* caps, int32_t dims, const double* total_rollouts, double mean_len,
                        gp_rollout_result* out, gp_rollout_entry* entries, int32_t* status) {
  NvtxRange nvtx("gp_solve_milp_batch");
  if (!ctx) return set_error(GP_INVALID, "null context");
  if (q < 0 || (q > 0 && (!configs || !cfg_off || !caps || !total_rollouts || !out || !entries || !status)))
    return set_error(GP_INVALID, "null argument");
  cudaSetDevice(ctx->device);
  std::vector<const gp_config*> cp(q);
  std::vector<int> nc(q);
  std::vector<const int32_t*> capp(q);
  std::vector<gp_rollout_entry*> ep(q);
  std::vector<int> rcs(q);
  for (int i = 0; i < q; ++i) {
    cp[i] = configs + cfg_off[i];
    nc[i] = cfg_off[i + 1] - cfg_off[i];
    capp[i] = caps + (size_t)i * dims;
    ep[i] = entries + cfg_off[i];
  }
  int rc = milp_batch(ctx, q, cp.data(), nc.data(), capp.data(), dims, total_rollouts, mean_len, out, ep.data(),
                      rcs.data());
  for (int i = 0; i < q; ++i) status[i] = rcs[i];
  return rc;
}

int gp_weight_sync_cost(gp_ctx* ctx, const int32_t* train, int32_t n_train, const int32_t* rollout,
                        int32_t n_rollout, const int32_t* entry_types, const int32_t* entry_replicas,
                        int32_t n_entries, int32_t window, double* out) {
  NvtxRange nvtx("gp_weight_sync_cost");
  if (!ctx) return set_error(GP_INVALID, "null context");
  cudaSetDevice(ctx->device);
  return weight_sync(ctx, train, n_train, rollout, n_rollout, entry_types, entry_replicas, n_entries,
                     window, out);
}

int gp_partition_candidates(gp_ctx* ctx, const gp_gamma* gamma, const gp_part_opts* opts, int32_t k,
                            gp_partition* out, int32_t* train_ids, int32_t* n_out) {
  NvtxRange nvtx("gp_partition_candidates");
  if (!ctx) return set_error(GP_INVALID, "null context");
  cudaSetDevice(ctx->device);
  return partition_candidates(ctx, gamma, opts, k, out, train_ids, n_out);
}

int gp_partition_objective(gp_ctx* ctx, const int32_t* train, int32_t n_train, double* objective,
                           double* fraction) {
  if (!ctx) return set_error(GP_INVALID, "null context");
  cudaSetDevice(ctx->device);
  return partition_objective(ctx, train, n_train, objective, fraction);
}

int gp_compute_fraction(gp_ctx* ctx, const int32_t* train, int32_t n_train, double* fraction) {
  if (!ctx) return set_error(GP_INVALID, "null context");
  cudaSetDevice(ctx->device);
  return compute_fraction(ctx, train, n_train, fraction);
}

void gp_default_sched_opts(gp_sched_opts* o) {
  std::memset(o, 0, sizeof *o);
  o->eta_override = -1;
  o->stable_iters = 20;
  o->iteration_cap = 200;
  o->stability_tol = 0.005;
  o->balance_tol = 0.02;
  o->interval_min = 1e-3;
  o->band_widen_step = 0.05;
  o->delta_cap = 64;
  o->expand_window = 1;
  o->candidate_width = 8;
  o->grid_probes = 15;
  o->train.max_stages_per_type = 4;
  o->train.device_granularity_limit = 16;
  o->rollout.max_stages = 4;
  o->exact_threshold = 12;
  o->restarts = 16;
  o->seed = 0x5eedULL;
  o->band_epsilon = 1e-9;
}

int gp_schedule(gp_ctx* ctx, const gp_sched_opts* opts, gp_schedule_result* out, int32_t* train_ids,
                int32_t* rollout_ids, int32_t* stage_devices, gp_config* entry_configs,
                gp_rollout_entry* entries, int32_t entry_cap, double* trace) {
  if (!ctx || !opts) return set_error(GP_INVALID, "null argument");
  cudaSetDevice(ctx->device);
  return schedule(ctx, opts, out, train_ids, rollout_ids, stage_devices, entry_configs, entries, entry_cap, trace);
}

int gp_ctx_set_memo(gp_ctx* ctx, int on) {
  if (!ctx) return set_error(GP_INVALID, "null context");
  ctx->memo = on != 0;
  if (!ctx->memo) train_memo_free(ctx);
  return GP_OK;
}

int gp_ctx_set_timing(gp_ctx* ctx, int on) {
  if (!ctx) return set_error(GP_INVALID, "null context");
  cudaSetDevice(ctx->device);
  for (auto& e : ctx->ev)
    if (!e) GP_CUDA(cudaEventCreate(&e));
  ctx->timing = on != 0;
  return GP_OK;
}

// Device time of the last gp_train_launch: stage tables (K2) and layout scan (K1 + finalize).
int gp_train_timing(gp_ctx* ctx, float* k2_ms, float* k1_ms) {
  if (!ctx || !ctx->timing) return set_error(GP_INVALID, "timing not enabled");
  GP_CUDA(cudaEventElapsedTime(k2_ms, ctx->ev[0], ctx->ev[1]));
  GP_CUDA(cudaEventElapsedTime(k1_ms, ctx->ev[1], ctx->ev[2]));
  return GP_OK;
}

void gp_ctx_io_bytes(gp_ctx* ctx, long long* h2d, long long* d2h, double* sum_stages) {
  *h2d = ctx->h2d_bytes;
  *d2h = ctx->d2h_bytes;
  *sum_stages = ctx->sum_stages;
}

// FP64 pipe throughput probe (bench.py roofline denominator): independent DADD chains.
__global__ void __launch_bounds__(256) k_fp64_peak(double* out, int iters, double y) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < iters; ++i) {
    a0 += y; a1 += y; a2 += y; a3 += y; a4 += y; a5 += y; a6 += y; a7 += y;
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == -1.0) out[0] = a0;
}

int gp_fp64_peak(gp_ctx* ctx, double* dadd_per_s) {
  if (!ctx) return set_error(GP_INVALID, "null context");
  cudaSetDevice(ctx->device);
  double* d = static_cast<double*>(ctx_scratch(ctx, 1 << 20));
  if (!d) return GP_CUDA_ERROR;
  cudaEvent_t a, b;
  GP_CUDA(cudaEventCreate(&a));
  GP_CUDA(cudaEventCreate(&b));
  const int blocks = ctx->num_sms * 8, iters = 1 << 14;
  k_fp64_peak<<<blocks, 256, 0, ctx->stream>>>(d, iters, 1e-300);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    GP_CUDA(cudaEventRecord(a, ctx->stream));
    k_fp64_peak<<<blocks, 256, 0, ctx->stream>>>(d, iters, 1e-300);
    GP_CUDA(cudaEventRecord(b, ctx->stream));
    GP_CUDA(cudaEventSynchronize(b));
    float ms;
    GP_CUDA(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *dadd_per_s = (double)blocks * 256 * iters * 8 / (best * 1e-3);
  return GP_OK;
}

}  // extern "C"
