// gp_internal.h — shared host/device definitions of the B200 plan-evaluation engine.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>
#include <cstdio>

#include <atomic>
#include <string>
#include <vector>

#include "../../include/gplan.h"

namespace gp {

// A double updated from several host threads (GPLAN_PROFILE statistics: per-device threads of
// the multi-GPU batches add to the same counters).
struct AtomicD {
  std::atomic<double> v{0.0};
  void operator+=(double x) {
    double cur = v.load(std::memory_order_relaxed);
    while (!v.compare_exchange_weak(cur, cur + x, std::memory_order_relaxed)) {
    }
  }
  operator double() const { return v.load(std::memory_order_relaxed); }
};

// Debug builds (-DGP_DEBUG_CHECKS, tools/build_variant.sh checks): bounds / invariant checks
// inside the kernels; a failing check prints its location and traps. (compute-sanitizer is
// not available on the GPU pool this engine was developed on.)
#ifdef GP_DEBUG_CHECKS
#define GP_CHECK(cond)                                                                          \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("GP_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                                \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define GP_CHECK(cond) \
  do {                 \
  } while (0)
#endif

// NVTX range for the lifetime of a scope (header-only NVTX 3: free unless a tool such as
// Nsight Systems / ncu --nvtx is attached). Marks the driver phases and the C ABI calls.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr double kInf = 1e30;       // inc/common.hpp:41
constexpr long long kSlowQueue = 1 << 21;  // deferred generic candidates per scan (overflow -> rescan)
constexpr double kActBytes = 2.0;   // src/cost_model.cpp:10
constexpr int kMaxPerRun = 4;       // K1 kernel instantiations support <= 4 blocks per type run
constexpr long long kFanoutMinLayouts = 20000000;  // below this a search stays on one GPU
constexpr long long kBatchSplitMinLayouts = 1000000000;  // a train batch below this stays on one GPU
constexpr long long kMilpSplitMinStates = 20000000;      // a MILP batch below this stays on one GPU

// Derived workload/calibration scalars, computed on the host exactly as the
// reference's inline accessors do (inc/workload.hpp:51-58) and passed by value.
struct Scalars {
  double P;             // params()
  double tokens;        // tokens_per_step()
  double mtl;           // mean_total_len()
  double tfpt_tokens;   // train_flops_per_token() * tokens
  double mbi;           // model_bytes_infer()
  double ifpt;          // infer_flops_per_token()
  double kvbpt;         // kv_bytes_per_token()
  double act_tok_h2;    // tokens * hidden * 2.0 (stage transfer numerator)
  double bpp_train, bpp_infer;
  double act_coeff, tp_coeff, grad_bpp;
  double stage_pen, sync_latency, reward;
  int L, H, mb, max_conc, batch;
  double mean_len;
};

// Per train-set block record (one contiguous block of a type run).
struct BlockRec {
  int start;        // offset into the canonical order
  int n;            // devices
  int type;
  int per_machine;  // max_devices_per_machine
  double flops;     // sequential fold of device flops (src/train_search.cpp:229-232)
  double lf_num;    // num_layers * flops (allocate_layers numerator)
  double cap_front; // hbm_capacity of devices.front()
  double beta_tp[4];  // min link within TP groups for tp = 1,2,4,8 (index 0 unused)
  double beta_dp[4];  // min link within DP groups (stride tp)
};

// Launch-parameter view of one train set (fits in the kernel param space).
struct TrainSpace {
  int R;                 // type runs
  int max_stages;        // min(L, R * max_per_run)
  int max_per_run;
  int n;                 // devices in the train set
  int len[GP_MAX_TYPES];
  int nc[GP_MAX_TYPES];        // cut count per run
  int kmax[GP_MAX_TYPES];      // min(max_per_run, len)
  int blk_off[GP_MAX_TYPES];   // first block index of run r
  int tin_off[GP_MAX_TYPES];   // offset of run r's (nc+2)^3 within-run transfer cube
  int tx_off[GP_MAX_TYPES];    // offset of the (r, r+1) cross-run transfer matrix
  int64_t cnt[GP_MAX_TYPES + 1][GP_MAX_STAGES + 1];  // completions of runs r.. with u used
  int64_t cntP[GP_MAX_TYPES + 1][GP_MAX_STAGES + 1]; // same over the prefix runs 0..R-2 only
  int n_suf;             // suffix table size (all (k, cuts) choices of the last run)
};

// One choice of the last type run (the "suffix" of a layout), in enumeration order:
// its block ids, its internal stage-transfer terms and the end of its first block.
struct __align__(16) SufEnt {
  int bi[4];
  double t[3];
  int k;
  int b1;  // end position of the first block
  int bl;  // start position of the last block
};

// Fast-path view of a suffix choice, valid when the layer-allocation total is the same
// for every layout of the train set (see k1_layout_scan_fast): the suffix stages'
// remainders in stable descending order and floor sum, and, per promotion count b (its top
// b stages get one extra layer) and per number d of zero-layer fix-up donations taken from
// it, its zero-stage count and its largest layer count (k2f_suffix_fast).
constexpr int kDonations = 4;  // fix-up donations tabulated (more -> generic fallback)
constexpr int kMsStride = 32;  // bytes per suffix choice in TrainTables::sf_ms

// K1-fast's per-choice tables of the MIDDLE run (the last of the prefix runs, R - 2): the
// prefix tables of a combination (front runs 0..R-3, middle choice) are the merge of the
// front's (built by the warp when the front changes) and this row (k2m_middle_rows).
struct __align__(16) MidRow {  // (a multiple of 16 bytes: copied to shared memory in 16-byte chunks)
  double2 pt[5][5];      // (max total, max compute) of its stages: top a1 promoted, d1 donations
  double R[4];           // remainders in stable descending order (-1 pad)
  double t[3];           // internal stage-transfer terms (0 for absent ones)
  signed char mp[5][5];  // largest layer count after d1 donations (-1: no donor left; L <= 127)
  unsigned char nz[5];   // zero-layer stages at promotion a1
  unsigned char k, b1, bl;  // blocks, end of the first block, start of the last block
  int fs;                // floor sum
  int bad;               // bit a1: a promoted stage would exceed L layers
};
static_assert(sizeof(MidRow) == 512, "MidRow is copied in 32 16-byte chunks, one per lane");

// Device-side training tables of one train set.
struct TrainTables {
  const int* ordered;
  // machine groups of the canonical order (consecutive devices on one machine): group of
  // each position, first position of each group (+ end), machine id of each group
  const int* mgrp;
  const int* gstart;
  const int* gmach;
  const double* mlinks;  // [M * M] or nullptr (device-level links)
  int M;
  const int* pos;        // per run: positions [0, cuts..., len], offsets = pos_off
  const BlockRec* blk;
  const double2* stage;  // [nblk * L] (total, compute); total = +inf => memory-infeasible
  const int8_t* opt;     // [nblk * L] chosen tp option index
  const double* tin;
  const double* tx;
  const double* fd_coef; // [S] = (double)(S-1) / micro_batches
  const SufEnt* suf;     // [n_suf]
  // fast path (constant allocation total), structure-of-arrays over the suffix choices so
  // that a warp's 32 consecutive choices are read with coalesced loads (k2f_suffix_fast):
  const double2* blk_sh;  // [nblk] per block (remainder, floor) of its layer share
  const int4* sf_hot;     // [n_suf] floor sum; zero-layer stage count at promotion b = 4 | k << 8 |
                          //   junction byte offset << 16; run-local block ids of the stages in
                          //   remainder order (desc, stage order among equals), one byte each
                          //   (255: none); zero-layer stage counts at b = 0..3, one byte each
  const double* sf_t;     // internal stage-transfer terms: (t0, t1)[n_suf] as double2, then t2[n_suf]
  const signed char* sf_ms;  // [n_suf][kMsStride]: largest layer count at (b, d donations), -1: none
  const double2* sf_st;   // [5 * (kDonations + 1)][n_suf]: (max total, max compute) at (b, d)
  const int* nzs_max;     // suffix stats: [0] most zero-layer stages of any suffix choice,
                          //   [1] kFsBias - smallest floor sum, [2] largest floor sum
  const MidRow* mid;       // [choices of run R - 2] middle-run rows (K1-fast, R >= 2)
  const unsigned long long* cntb_mid;  // [choices of run R - 2][cw] rank counts of the last run's
                                       //   blocks among the middle remainders (bytes, 8 per word)
  int cw;                    // words per cntb_mid row
  int n_mid;                 // rows of mid
  int pos_off[GP_MAX_TYPES];
};

struct Best {
  double cost;
  long long rank;
  long long feasible;
};

__host__ __device__ inline int blk_index(int nc, int a, int b) {
  // blocks (a, b), 0 <= a < b <= nc+1, row-major by a
  return a * (nc + 1) - (a * (a - 1)) / 2 + (b - a - 1);
}
__host__ __device__ inline int64_t binom_small(int n, int j) {
  switch (j) {
    case 0: return 1;
    case 1: return n > 0 ? n : 0;
    case 2: return n > 1 ? (int64_t)n * (n - 1) / 2 : 0;
    case 3: return n > 2 ? (int64_t)n * (n - 1) * (n - 2) / 6 : 0;
  }
  return 0;
}

}  // namespace gp

// Engine context (opaque in the C ABI).
struct gp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  // cluster
  int N = 0, T = 0, M = 0;
  std::vector<int> h_type, h_machine;
  std::vector<double> h_flops, h_hbm_bw, h_hbm_cap, h_tflops, h_thbm, h_tcap, h_ceff, h_ioeff;
  int* d_type = nullptr;
  int* d_machine = nullptr;
  double* d_flops = nullptr;
  double* d_hbm_bw = nullptr;
  double* d_hbm_cap = nullptr;
  double* d_links = nullptr;
  // machine-pair link table, set when every link(a != b) depends only on (machine(a),
  // machine(b)) — certified at context creation; K2a/K2b then take minima over machines
  double* d_mlinks = nullptr;
  double* d_ceff = nullptr;
  double* d_ioeff = nullptr;
  double* d_tflops = nullptr;
  double* d_thbm = nullptr;
  double* d_tcap = nullptr;
  gp::Scalars sc{};
  gp_workload work{};
  gp_calib calib{};
  // grow-only device scratch, one arena per subsystem (0 train, 1 rollout, 2 partition)
  void* scratch_arena[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t scratch_arena_bytes[4] = {0, 0, 0, 0};
  void* h_pinned = nullptr;
  size_t h_pinned_bytes = 0;
  int num_sms = 148;
  // kernel launches issued by this context (bench.py's gpu_launches claim)
  long long launches = 0;
  // prepared train set (train.cu), cached MILP lattice table (rollout.cu)
  void* train_state = nullptr;
  void* milp_cache = nullptr;
  void* part_cache[2] = {nullptr, nullptr};  // partition unit tables per granularity (partition.cu)
  // K1-fast's deferred generic candidates: [0] = count, then keys (train.cu)
  unsigned long long* d_slow = nullptr;
  // train_batch runs its train sets on kTrainLanes streams (each with its own queue)
  static constexpr int kTrainLanes = 4;
  cudaStream_t lane[kTrainLanes] = {};
  unsigned long long* d_slow_lane[kTrainLanes] = {};
  cudaEvent_t ev_lane[kTrainLanes + 1] = {};
  // constrained_search results per train set, window-independent (train.cu TrainMemo)
  void* train_memo = nullptr;
  bool memo = true;
  // peer contexts on other GPUs (gp_ctx_create_multi): constrained_search fans out over them
  std::vector<gp_ctx*> peers;
  // multi-device contexts: an auxiliary context on the last device, on which the native
  // driver computes the next iteration's candidate partitions while the current iteration's
  // evaluation batch runs (schedule.cu)
  gp_ctx* aux = nullptr;
  // optional device timing of the train phases (bench.py): events around K2 and K1
  bool timing = false;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  // host<->device bytes moved by API calls (bench.py's e2e accounting)
  long long h2d_bytes = 0, d2h_bytes = 0;
  // sum over the prepared train set's layouts of the stage count (roofline accounting)
  double sum_stages = 0;
};

namespace gp {
int set_error(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
enum { kArenaTrain = 0, kArenaRollout = 1, kArenaPartition = 2, kArenaMisc = 3 };
void* ctx_scratch(gp_ctx* ctx, size_t bytes, int arena = kArenaMisc);
void* ctx_pinned(gp_ctx* ctx, size_t bytes);
}  // namespace gp

#define GP_CUDA(call)                                          \
  do {                                                         \
    cudaError_t e_ = (call);                                   \
    if (e_ != cudaSuccess) return gp::cuda_fail(e_, #call);    \
  } while (0)
