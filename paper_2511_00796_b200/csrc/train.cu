// train.cu — sm_100a kernels for the training-side hot loop:
//   constrained_search (src/train_search.cpp:218-275) over the layout space of
//   enumerate_block_lists (src/train_search.cpp:126-142), scored with
//   train_stage_cost / train_cost_breakdown / mem_cumsum_train
//   (src/cost_model.cpp:57-126,198-207).
//
// Design:
//   K2a  block_stats   one CTA per contiguous block of a type run: sequential
//                      FLOPS fold, per-machine count, exact min-link over the TP
//                      (chunked) and DP (strided) groups of every tp option.
//   K2b  transfers     one warp per adjacent block pair: exact min-link over the
//                      block x block rectangle -> stage-transfer term.
//   K2c  stage_table   one thread per (block, layer_count): memory filter +
//                      comm-minimal (tp, dp) pick -> (total, compute).
//   K1   layout_scan   persistent grid; each thread unranks a chunk start of the
//                      layout rank space and walks the chunk with an odometer
//                      (no plan list is materialised); allocate_layers + table
//                      gathers + fill/drain + transfers; lexicographic
//                      (cost, rank) argmin via warp shuffles -> CTA -> grid.
//   K1f  finalize      reduce CTA partials, decode the winning rank.
// Every fp64 expression keeps the reference's association order; the library
// is compiled with --fmad=false, so results are bit-identical to the CPU.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <unordered_map>
#include <mutex>
#include <thread>
#include <array>

#include "gp_internal.h"

namespace gp {

struct TrainOut {
  Best best;
  long long nm_b0;       // near-minimum summary of the scanned range (NearMin), keys decoded to ranks
  long long nm_rank[3];
  int n_stages;
  int overflow;  // K1-fast's deferred queue overflowed: the host rescans with the generic K1
  int first[GP_MAX_STAGES];
  int count[GP_MAX_STAGES];
  int tp[GP_MAX_STAGES];
  int dp[GP_MAX_STAGES];
  int layers[GP_MAX_STAGES];
};

struct BlockMeta {
  int run, a, b, start_global;
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = dmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// CTA-wide min; every thread gets the result.
__device__ double block_min(double v, double* sm) {
  v = warp_min(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  double r = lane < nw ? sm[lane] : kInf;
  r = warp_min(r);
  return r;
}


// Window-independent argmin summary. The reference scores a layout by
// cost = window * per_step (src/train_search.cpp, oracle/oracle.c:337) and keeps the first
// rank of minimal cost. fl(window * x) is monotone in x, so the minimal cost is
// fl(window * x_min), and a layout ties with it only if fl(window * x) == fl(window * x_min),
// which needs x < x_min + 2 ulp(x_min) (|w x - w x_min| < ulp(w x_min) <= 2 w ulp(x_min)).
// Positive doubles order like their bit patterns, so it suffices to keep, for the three bit
// patterns b0, b0+1, b0+2 above the smallest per-step time b0, the first key reaching each:
// the argmin for ANY window is then the first key among the patterns whose scaled cost equals
// the smallest one. One scan therefore answers every window of the scheduler's passes.
struct NearMin {
  long long b0;      // bit pattern of the smallest feasible per-step time (kInfBits when none)
  long long key[3];  // first key whose per-step time has bit pattern b0 + i (LLONG_MAX if none)
  long long feasible;
};

constexpr long long kInfBits = 0x7ff0000000000000LL;

__host__ __device__ __forceinline__ void nm_init(NearMin& m) {
  m.b0 = kInfBits;
  m.key[0] = m.key[1] = m.key[2] = LLONG_MAX;
  m.feasible = 0;
}

// key of pattern b0 + j (selects, not a dynamic index: keeps summaries in registers)
__host__ __device__ __forceinline__ long long nm_at(const NearMin& m, long long j) {
  return j == 0 ? m.key[0] : j == 1 ? m.key[1] : j == 2 ? m.key[2] : LLONG_MAX;
}

// m := merge(m, o); both summaries are exact for disjoint key sets.
__host__ __device__ __forceinline__ void nm_merge(NearMin& m, const NearMin& o) {
  m.feasible += o.feasible;
  const long long base = o.b0 < m.b0 ? o.b0 : m.b0;
  const long long dm = m.b0 - base, dn = o.b0 - base;
  long long k[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const long long a = nm_at(m, i - dm), b = nm_at(o, i - dn);
    k[i] = a < b ? a : b;
  }
  m.b0 = base;
#pragma unroll
  for (int i = 0; i < 3; ++i) m.key[i] = k[i];
}

// First key among the near-minimum patterns whose window-scaled cost is the minimum.
__host__ __device__ __forceinline__ long long nm_winner(const NearMin& m, int window, double& cost) {
  long long bits = m.b0;
  double x0;
  memcpy(&x0, &bits, sizeof x0);
  cost = window * x0;
  long long win = LLONG_MAX;
  for (int i = 0; i < 3; ++i) {
    if (m.key[i] == LLONG_MAX) continue;
    bits = m.b0 + i;
    double x;
    memcpy(&x, &bits, sizeof x);
    if (window * x == cost && m.key[i] < win) win = m.key[i];
  }
  return win;
}

// ---------------------------------------------------------------- K2a blocks
// min_link_within_groups (src/cost_model.cpp:12-36), exact, for every option.
// CTA-cooperative body: block `bidx` of the set (also run by the fused small-set kernel).
__device__ __forceinline__ void k2a_body(int bidx, const int* __restrict__ ordered,
                                         const BlockMeta* __restrict__ meta, const int* __restrict__ pos,
                                         const TrainTables& tb, BlockRec* __restrict__ out,
                                         const int* __restrict__ dtype, const int* __restrict__ dmachine,
                                         const double* __restrict__ dflops, const double* __restrict__ dcap,
                                         const double* __restrict__ links, int N, int L, int mb,
                                         double* fd_coef, double2* __restrict__ blkf) {
  __shared__ double red[32];
  __shared__ BlockRec rec;
  const BlockMeta m = meta[bidx];
  const int* P = pos + tb.pos_off[m.run];
  const int start = m.start_global + P[m.a];
  const int n = P[m.b] - P[m.a];
  const int* dev = ordered + start;
  if (threadIdx.x == 0) {
    rec.start = start;
    rec.n = n;
    rec.type = dtype[dev[0]];
    double f = 0;
    int best = 0, run = 0;
    for (int i = 0; i < n; ++i) {
      f += dflops[dev[i]];
      run = (i > 0 && dmachine[dev[i]] == dmachine[dev[i - 1]]) ? run + 1 : 1;
      best = run > best ? run : best;
    }
    rec.flops = f;
    rec.lf_num = L * f;
    rec.per_machine = best;
    rec.cap_front = dcap[dev[0]];
    for (int o = 0; o < 4; ++o) rec.beta_tp[o] = rec.beta_dp[o] = kInf;
  }
  if (bidx == 0)
    for (int S = threadIdx.x; S <= GP_MAX_STAGES; S += blockDim.x)
      fd_coef[S] = S > 0 ? static_cast<double>(S - 1) / mb : 0.0;
  __syncthreads();
  const int per_machine = rec.per_machine;
#pragma unroll 1
  for (int o = 0; o < 4; ++o) {
    const int tp = 1 << o;
    if (tp > per_machine || n % tp != 0) continue;  // tp_dp_options (src/train_search.cpp:74-93)
    const int dp = n / tp;
    if (tb.mlinks) {  // machine-structured links: minima over machine-group pairs
      // a pair (earlier, later) of distinct devices has link mlinks[m(earlier)][m(later)];
      // groups are in canonical (machine) order, so earlier devices sit in groups <= later
      if (tp > 1) {
        double mn = kInf;
        for (int c = threadIdx.x; c < n / tp; c += blockDim.x) {
          const int p0 = start + c * tp, p1 = p0 + tp;  // chunk [p0, p1)
          const int ga = tb.mgrp[p0], gb = tb.mgrp[p1 - 1];
          for (int g = ga; g <= gb; ++g)
            for (int h = g; h <= gb; ++h) {
              if (g == h) {
                const int cnt = min(p1, tb.gstart[g + 1]) - max(p0, tb.gstart[g]);
                if (cnt < 2) continue;
              }
              mn = dmin(mn, tb.mlinks[(size_t)tb.gmach[g] * tb.M + tb.gmach[h]]);
            }
        }
        mn = block_min(mn, red);
        if (threadIdx.x == 0) rec.beta_tp[o] = mn;
      }
      if (dp > 1) {  // stride-tp groups: devices start + g + i*tp, i < dp
        double mn = kInf;
        const int ga = tb.mgrp[start], K = tb.mgrp[start + n - 1] - ga + 1;
        auto cnt = [&](int g, int k) {  // devices of stride group g on machine group k
          const int x0 = tb.gstart[k] - start - g, x1 = tb.gstart[k + 1] - start - g;
          const int lo = x0 <= 0 ? 0 : (x0 + tp - 1) / tp;
          const int hi = x1 <= 0 ? 0 : min(dp, (x1 + tp - 1) / tp);
          return hi > lo ? hi - lo : 0;
        };
        for (int idx = threadIdx.x; idx < tp * K * K; idx += blockDim.x) {
          const int g = idx / (K * K), rem = idx % (K * K);
          const int k = ga + rem / K, k2 = ga + rem % K;
          if (k2 < k) continue;
          const int c1 = cnt(g, k);
          if (k == k2 ? c1 < 2 : (c1 == 0 || cnt(g, k2) == 0)) continue;
          mn = dmin(mn, tb.mlinks[(size_t)tb.gmach[k] * tb.M + tb.gmach[k2]]);
        }
        mn = block_min(mn, red);
        if (threadIdx.x == 0) rec.beta_dp[o] = mn;
      }
      continue;
    }
    if (tp > 1) {  // consecutive chunks of tp devices
      double mn = kInf;
      const int pairs_per = tp * (tp - 1) / 2;
      const int total = (n / tp) * pairs_per;
      for (int p = threadIdx.x; p < total; p += blockDim.x) {
        const int g = p / pairs_per;
        int q = p - g * pairs_per, i = 0;
        while (q >= tp - 1 - i) {
          q -= tp - 1 - i;
          ++i;
        }
        const int j = i + 1 + q;
        mn = dmin(mn, links[(size_t)dev[g * tp + i] * N + dev[g * tp + j]]);
      }
      mn = block_min(mn, red);
      if (threadIdx.x == 0) rec.beta_tp[o] = mn;
    }
    if (dp > 1) {  // stride-tp groups of dp devices
      double mn = kInf;
      const long long sq = (long long)dp * dp;
      for (long long p = threadIdx.x; p < sq; p += blockDim.x) {
        const int i = (int)(p / dp), j = (int)(p - (long long)i * dp);
        if (i >= j) continue;
        for (int g = 0; g < tp; ++g)
          mn = dmin(mn, links[(size_t)dev[i * tp + g] * N + dev[j * tp + g]]);
      }
      mn = block_min(mn, red);
      if (threadIdx.x == 0) rec.beta_dp[o] = mn;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[bidx] = rec;
    blkf[bidx] = make_double2(rec.flops, rec.lf_num);  // K1's (flops, L*f) view
  }
  __syncthreads();  // rec is reused by the next block of a fused loop
}

__global__ void __launch_bounds__(256) k2a_block_stats(const int* __restrict__ ordered,
                                                       const BlockMeta* __restrict__ meta,
                                                       const int* __restrict__ pos,
                                                       TrainTables tb, BlockRec* __restrict__ out,
                                                       const int* __restrict__ dtype,
                                                       const int* __restrict__ dmachine,
                                                       const double* __restrict__ dflops,
                                                       const double* __restrict__ dcap,
                                                       const double* __restrict__ links, int N,
                                                       int L, int mb, double* fd_coef,
                                                       double2* __restrict__ blkf) {
  k2a_body(blockIdx.x, ordered, meta, pos, tb, out, dtype, dmachine, dflops, dcap, links, N, L, mb, fd_coef, blkf);
}

// ------------------------------------------------------------ K2b transfers
// min_link_between (src/cost_model.cpp:38-47) over adjacent blocks; one warp per item.
// item = (run, a, b, c): within-run blocks [a,b) -> [b,c); c < 0 marks a cross-run item
// (run r's block [a, nc+1) -> run r+1's block [0, -c)).
// warp body: item `warp` of the set
__device__ __forceinline__ void k2b_body(int warp, int lane, const int* __restrict__ ordered,
                                         const int4* __restrict__ items, const int* __restrict__ pos,
                                         const TrainTables& tb, const TrainSpace& sp,
                                         const int* __restrict__ run_start, const double* __restrict__ links,
                                         int N, double numer, double* tin, double* tx) {
  const int4 it = items[warp];
  const int r = it.x;
  const int* P = pos + tb.pos_off[r];
  int s1, n1, s2, n2;
  if (it.w >= 0) {
    s1 = run_start[r] + P[it.y];
    n1 = P[it.z] - P[it.y];
    s2 = run_start[r] + P[it.z];
    n2 = P[it.w] - P[it.z];
  } else {
    const int* P2 = pos + tb.pos_off[r + 1];
    s1 = run_start[r] + P[it.y];
    n1 = sp.len[r] - P[it.y];
    s2 = run_start[r + 1];
    n2 = P2[-it.w];
  }
  double mn = kInf;
  if (tb.mlinks) {  // machine-structured links: the minimum over the machine pairs
    const int ga = tb.mgrp[s1], gb = tb.mgrp[s1 + n1 - 1], ha = tb.mgrp[s2], hb = tb.mgrp[s2 + n2 - 1];
    const int k2 = hb - ha + 1, tot = (gb - ga + 1) * k2;
    for (int p = lane; p < tot; p += 32) {
      const int g = ga + p / k2, h = ha + p % k2;
      mn = dmin(mn, tb.mlinks[(size_t)tb.gmach[g] * tb.M + tb.gmach[h]]);
    }
  } else {
    const long long tot = (long long)n1 * n2;
    for (long long p = lane; p < tot; p += 32) {
      const int i = (int)(p / n2), j = (int)(p - (long long)i * n2);
      mn = dmin(mn, links[(size_t)ordered[s1 + i] * N + ordered[s2 + j]]);
    }
  }
  mn = warp_min(mn);
  if (lane == 0) {
    // tokens * hidden * kActivationBytes / beta; skipped entirely when tokens <= 0
    const double t = numer > 0 ? numer / mn : 0.0;
    if (it.w >= 0) {
      const int e = sp.nc[r] + 2;
      tin[sp.tin_off[r] + ((size_t)it.y * e + it.z) * e + it.w] = t;
    } else {
      const int e2 = sp.nc[r + 1] + 2;
      tx[sp.tx_off[r] + (size_t)it.y * e2 + (-it.w)] = t;
    }
  }
}

__global__ void __launch_bounds__(256) k2b_transfers(const int* __restrict__ ordered,
                                                     const int4* __restrict__ items, int n_items,
                                                     const int* __restrict__ pos, TrainTables tb,
                                                     TrainSpace sp, const int* __restrict__ run_start,
                                                     const double* __restrict__ links, int N,
                                                     double numer, double* tin, double* tx) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= n_items) return;
  k2b_body(warp, threadIdx.x & 31, ordered, items, pos, tb, sp, run_start, links, N, numer, tin, tx);
}

// ------------------------------------------------------------ K2c stage table
// Per (block, layer_count): the option loop of constrained_search
// (src/train_search.cpp:241-265) with mem_cumsum_train and train_stage_cost.
// One (tp, dp) option of a stage with lc layers (src/train_search.cpp:241-258 with
// tp_dp_options :74-93, mem_cumsum_train src/cost_model.cpp:198-207, train_stage_cost
// :57-91). False when the option is not offered or exceeds the block's memory.
__device__ __forceinline__ bool stage_option(const BlockRec& b, int lc, int o, const Scalars& sc,
                                             double ceff, double& compute, double& tp_comm,
                                             double& dp_comm) {
  const int tp = 1 << o;
  if (tp > b.per_machine || b.n % tp != 0) return false;
  const int dp = b.n / tp;
  const double lf = static_cast<double>(lc) / sc.L;  // layer_frac (total_layers == num_layers)
  const double weight = sc.P * lf * sc.bpp_train / tp;
  const double tpm = sc.tokens / dp / sc.mb;
  const double act = sc.act_coeff * tpm * sc.H * kActBytes * lc / tp;
  const double need_gb = (weight + act) / 1e9;
  if (need_gb * 1e9 > b.cap_front) return false;
  compute = sc.tfpt_tokens * lf / (ceff * b.flops);
  tp_comm = 0;
  dp_comm = 0;
  if (tp > 1 && sc.tokens > 0) {
    const double prt = sc.tokens / dp;
    const double vol = sc.tp_coeff * lc * prt * sc.H * kActBytes * 2.0 * (tp - 1) / tp;
    tp_comm = vol / b.beta_tp[o];
  }
  if (dp > 1) {
    const double shard = sc.P * lf * sc.grad_bpp / tp;
    const double vol = 2.0 * shard * (dp - 1) / dp;
    dp_comm = vol / b.beta_dp[o];
  }
  return true;
}

// mode 0 (constrained_search): per (block, layers) the comm-minimal memory-feasible option
// (strict <, tp ascending). mode 1 (product space, enumerate_train_candidates): the option of
// minimal TrainStageCost::total() — the value the product-space argmin reaches per stage.
__device__ __forceinline__ void k2c_body(long long idx, const BlockRec* __restrict__ blk, const Scalars& sc,
                                         const double* __restrict__ ceff, int mode, double2* __restrict__ stage,
                                         int8_t* __restrict__ opt) {
  const int bi = (int)(idx / sc.L);
  const int lc = (int)(idx - (long long)bi * sc.L) + 1;
  const BlockRec& b = blk[bi];
  double best_key = -1, best_total = 0, compute = 0;
  int best_o = -1;
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    double cmp, tp_comm, dp_comm;
    if (!stage_option(b, lc, o, sc, ceff[b.type], cmp, tp_comm, dp_comm)) continue;
    compute = cmp;  // option-independent
    const double total = cmp + tp_comm + dp_comm;
    const double key = mode == 0 ? tp_comm + dp_comm : total;
    if (best_key < 0 || key < best_key) {
      best_key = key;
      best_total = total;
      best_o = o;
    }
  }
  if (best_o < 0) {  // still report compute (option-independent) for the fill/drain term
    const double lf = static_cast<double>(lc) / sc.L;
    compute = sc.tfpt_tokens * lf / (ceff[b.type] * b.flops);
  }
  double2 e;
  // TrainStageCost::total(); +inf marks "no memory-feasible option" so that the layout
  // maximum becomes +inf and the layout is rejected without a per-stage test in K1
  e.x = best_o < 0 ? __longlong_as_double(0x7ff0000000000000LL) : best_total;
  e.y = compute;
  stage[idx] = e;
  opt[idx] = (int8_t)best_o;
}

__global__ void __launch_bounds__(256) k2c_stage_table(const BlockRec* __restrict__ blk, int nblk,
                                                       Scalars sc, const double* __restrict__ ceff,
                                                       int mode, double2* __restrict__ stage,
                                                       int8_t* __restrict__ opt) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)nblk * sc.L) return;
  k2c_body(idx, blk, sc, ceff, mode, stage, opt);
}


// --------------------------------------------------------- K2d suffix table
// One entry per choice (k, cuts) of type run r (the LAST run for the generic scan, the
// inner run for K1-fast), in run_compositions order (src/train_search.cpp:53-72, k
// ascending): block ids, internal transfers, first-block end and last-block start.
__device__ __forceinline__ void k2d_body(int i, const int4* __restrict__ choices, const TrainSpace& sp,
                                         const double* __restrict__ tin, SufEnt* __restrict__ suf, int r) {
  const int nc = sp.nc[r], e = nc + 2;
  const int4 c = choices[i];  // (k, b1, b2, b3) position-index boundaries
  const int k = c.x;
  int b[5] = {0, c.y, c.z, c.w, 0};
  b[k] = nc + 1;
  SufEnt out;
#pragma unroll
  for (int j = 0; j < 4; ++j) out.bi[j] = j < k ? sp.blk_off[r] + blk_index(nc, b[j], b[j + 1]) : 0;
#pragma unroll
  for (int j = 0; j < 3; ++j)
    out.t[j] = j + 1 < k ? tin[sp.tin_off[r] + ((size_t)b[j] * e + b[j + 1]) * e + b[j + 2]] : 0.0;
  out.k = k;
  out.b1 = b[1];
  out.bl = b[k - 1];
  suf[i] = out;
}

__global__ void k2d_suffix_table(const int4* __restrict__ choices, int n, TrainSpace sp,
                                 const double* __restrict__ tin, SufEnt* __restrict__ suf, int r) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  k2d_body(i, choices, sp, tin, suf, r);
}

// ------------------------------------------------------------- K1 layout scan
// Rank space = concatenation over prefixes p (choices of runs 0..R-2, in
// enumeration order) of the suffix choices s < ns(u_p) of the last run. A warp
// owns a range of prefixes; its lanes stride over the suffixes of each prefix.
// The prefix's stage data are warp-uniform; per lane only the suffix differs.
template <int R>
struct Prefix {
  int k[R > 1 ? R - 1 : 1];
  int b[R > 1 ? R - 1 : 1][kMaxPerRun + 1];
  int u;
  long long base;  // rank of the prefix's first layout (generic scan: original run order)
  int ci[R > 1 ? R - 1 : 1];  // choice index of each prefix run (run_compositions order)
};

// positions b[1..m] (1-based cut indices, increasing) of the q-th m-subset of nc cuts in
// lexicographic order (run_compositions, src/train_search.cpp:53-72)
__host__ __device__ __forceinline__ void comb_unrank(int nc, int m, long long q, int* b) {
  int v = 0;
#pragma unroll
  for (int j = 1; j < kMaxPerRun; ++j) {
    if (j <= m) {
      while (true) {
        const long long cc = binom_small(nc - v - 1, m - j);
        if (q < cc) break;
        q -= cc;
        ++v;
      }
      b[j] = v + 1;
      ++v;
    }
  }
}

// Decode prefix index x over runs 0..R-2 (Enumerator::recurse order). Returns the
// full-space rank of the prefix's first layout (its base).
template <int R>
__host__ __device__ __forceinline__ long long prefix_decode(const TrainSpace& sp, long long x,
                                                            Prefix<R>& P) {
  int u = 0;
  long long base = 0;
#pragma unroll
  for (int r = 0; r + 1 < R; ++r) {
    const int nc = sp.nc[r];
    const int rem_runs = R - 1 - r;
    int cidx = 0;
    for (int k = 1; k <= sp.kmax[r]; ++k) {
      if (u + k + rem_runs > sp.max_stages) break;
      const long long c = binom_small(nc, k - 1);
      const long long subP = sp.cntP[r + 1][u + k];
      const long long sub = sp.cnt[r + 1][u + k];
      if (x < c * subP) {
        long long q = x / subP;
        x -= q * subP;
        base += q * sub;
        P.k[r] = k;
        P.ci[r] = cidx + (int)q;
        comb_unrank(nc, k - 1, q, P.b[r]);
#pragma unroll
        for (int j = 1; j <= kMaxPerRun; ++j)
          if (j == k) P.b[r][j] = nc + 1;
        P.b[r][0] = 0;
        u += k;
        break;
      }
      x -= c * subP;
      base += c * sub;
      cidx += (int)c;
    }
  }
  P.u = u;
  P.base = base;
  return base;
}

// rank -> (prefix runs 0..R-2 into P, index s among the last run's choices): the inverse of
// the enumeration order (Enumerator::recurse, src/train_search.cpp:95-124).
template <int R>
__host__ __device__ __forceinline__ void rank_decode(const TrainSpace& sp, long long rank, Prefix<R>& P,
                                                     long long& s) {
  int u = 0;
  s = 0;
  P.base = 0;
  for (int r = 0; r < R; ++r) {
    const int nc = sp.nc[r], rem_runs = R - 1 - r;
    long long sidx = 0;
    for (int k = 1; k <= sp.kmax[r]; ++k) {
      if (u + k + rem_runs > sp.max_stages) break;
      const long long c = binom_small(nc, k - 1), sub = sp.cnt[r + 1][u + k];
      if (rank < c * sub) {
        const long long q = rank / sub;
        rank -= q * sub;
        if (r + 1 < R) {
          P.k[r] = k;
          comb_unrank(nc, k - 1, q, P.b[r]);
          for (int j = 1; j <= kMaxPerRun; ++j)
            if (j == k) P.b[r][j] = nc + 1;
          P.b[r][0] = 0;
        } else {
          s = sidx + q;
        }
        u += k;
        break;
      }
      rank -= c * sub;
      sidx += c;
    }
    if (r + 2 == R) P.u = u;
  }
  if (R == 1) P.u = 0;
}

// Next prefix in enumeration order (odometer over runs 0..R-2).
template <int R>
__device__ __forceinline__ void prefix_advance(const TrainSpace& sp, Prefix<R>& P) {
  P.base += sp.cnt[R - 1][P.u];
  bool carry = true;
  int used[R > 1 ? R - 1 : 1];
  int acc = 0;
#pragma unroll
  for (int r = 0; r + 1 < R; ++r) {
    used[r] = acc;
    acc += P.k[r];
  }
#pragma unroll
  for (int rr = R - 2; rr >= 0; --rr) {
    if (carry) {
      const int nc = sp.nc[rr];
      const int m = P.k[rr] - 1;
      int jf = 0;
#pragma unroll
      for (int j = kMaxPerRun - 1; j >= 1; --j)
        if (jf == 0 && j <= m && P.b[rr][j] < nc - (m - j)) jf = j;
      bool ok = false;
      if (jf) {
#pragma unroll
        for (int j = 1; j < kMaxPerRun; ++j) {
          if (j == jf) P.b[rr][j] += 1;
          else if (j > jf && j <= m) P.b[rr][j] = P.b[rr][j - 1] + 1;
        }
        P.ci[rr]++;
        ok = true;
      } else if (P.k[rr] < sp.kmax[rr] && used[rr] + P.k[rr] + 1 + (R - 1 - rr) <= sp.max_stages &&
                 nc >= P.k[rr]) {
        const int k = ++P.k[rr];
#pragma unroll
        for (int j = 1; j <= kMaxPerRun; ++j) {
          if (j < k) P.b[rr][j] = j;
          else if (j == k) P.b[rr][j] = nc + 1;
        }
        P.ci[rr]++;
        ok = true;
      }
      if (ok) {
        carry = false;
#pragma unroll
        for (int r2 = rr + 1; r2 + 1 < R; ++r2) {
          P.k[r2] = 1;
          P.b[r2][1] = sp.nc[r2] + 1;
          P.ci[r2] = 0;
        }
      }
    }
  }
  int u = 0;
#pragma unroll
  for (int r = 0; r + 1 < R; ++r) u += P.k[r];
  P.u = u;
}

// Warp-uniform data of one prefix.
template <int R>
struct PrefixData {
  static constexpr int NP = (R - 1) * kMaxPerRun;
  int bi[NP > 0 ? NP : 1];
  double lfn[NP > 0 ? NP : 1];
  bool act[NP > 0 ? NP : 1];
  double total;      // left fold of the prefix stages' FLOPS (allocate_layers total, first part)
  double transfers;  // left fold of the prefix-internal stage transfers
  int a_last;        // start position of the prefix's last block (junction transfer)
  int u;             // prefix stage count
};

template <int R>
__device__ __forceinline__ void prefix_data(const TrainSpace& sp, const TrainTables& tb,
                                            const double2* __restrict__ blkf, const Prefix<R>& P,
                                            PrefixData<R>& D) {
  D.total = 0.0;
  D.transfers = 0.0;
  D.a_last = 0;
  D.u = P.u;
#pragma unroll
  for (int r = 0; r + 1 < R; ++r) {
#pragma unroll
    for (int j = 0; j < kMaxPerRun; ++j) {
      const int q = r * kMaxPerRun + j;
      D.act[q] = j < P.k[r];
      D.bi[q] = 0;
      D.lfn[q] = 0;
      if (D.act[q]) {
        D.bi[q] = sp.blk_off[r] + blk_index(sp.nc[r], P.b[r][j], P.b[r][j + 1]);
        const double2 fl = blkf[D.bi[q]];
        D.total += fl.x;
        D.lfn[q] = fl.y;
        if (j + 1 < P.k[r]) {
          const int e = sp.nc[r] + 2;
          D.transfers += tb.tin[sp.tin_off[r] + ((size_t)P.b[r][j] * e + P.b[r][j + 1]) * e +
                                P.b[r][j + 2 <= kMaxPerRun ? j + 2 : kMaxPerRun]];
        } else if (r + 2 < R) {
          const int e2 = sp.nc[r + 1] + 2;
          D.transfers += tb.tx[sp.tx_off[r] + (size_t)P.b[r][j] * e2 + P.b[r + 2 < R ? r + 1 : r][1]];
        } else {
          D.a_last = P.b[r][j];
        }
      }
    }
  }
}

// a / b correctly rounded, given y = RN(1/b): Markstein's theorem (q within one ulp,
// y within half an ulp -> one FMA residual correction yields RN(a/b)); operands are
// positive normals far from the exponent limits. Pinned by tests/test_engine_train.py.
__device__ __forceinline__ double div_rn_recip(double a, double b, double y) {
  const double q = __dmul_rn(a, y);
  const double r = __fma_rn(-q, b, a);
  return __fma_rn(r, y, q);
}

// Score (prefix, suffix). Returns false when some stage has no memory-feasible option.
template <int R, bool DECODE>
__device__ __forceinline__ bool eval_layout(const TrainSpace& sp, const TrainTables& tb,
                                            const double2* __restrict__ blkf, int L,
                                            const PrefixData<R>& D, const SufEnt& e, double& per_step,
                                            int* out_lay, int* out_bi) {
  constexpr int NP = (R - 1) * kMaxPerRun;
  constexpr int NS = NP + kMaxPerRun;
  // Prefix fields are re-read from the warp's shared-memory copy where they are used
  // (volatile: keeps them out of registers across the phases below).
  auto vbi = [&](int q) { return *(const volatile int*)&D.bi[q]; };
  auto vlfn = [&](int q) { return *(const volatile double*)&D.lfn[q]; };
  bool act[NS];
  int lay[NS];
  double rem[NS];
  double total = D.total;
#pragma unroll
  for (int q = 0; q < NP; ++q) act[q] = D.act[q];
  const int k = e.k;
  double lfn_s[kMaxPerRun];
#pragma unroll
  for (int j = 0; j < kMaxPerRun; ++j) {
    const int q = NP + j;
    act[q] = j < k;
    lfn_s[j] = 0;
    if (act[q]) {
      const double2 fl = blkf[e.bi[j]];
      total += fl.x;  // allocate_layers total: left fold in stage order
      lfn_s[j] = fl.y;
    }
  }
  const int S = D.u + k;
  const double y = 1.0 / total;
  int assigned = 0;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    const double share = div_rn_recip(q < NP ? vlfn(q) : lfn_s[q - NP], total, y);  // L * f / total
    lay[q] = static_cast<int>(share);
    rem[q] = act[q] ? share - lay[q] : -1.0;  // remainder >= +0 for active slots
    assigned += act[q] ? lay[q] : 0;
  }
  // std::stable_sort of remainders (desc) -> position of each slot; equal remainders
  // keep slot (stage) order. One DSETP + two predicated adds per pair.
  int pos[NS];
#pragma unroll
  for (int q = 0; q < NS; ++q) pos[q] = 0;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
#pragma unroll
    for (int q2 = q + 1; q2 < NS; ++q2) {
      asm("{\n\t.reg .pred p;\n\tsetp.ge.f64 p, %2, %3;\n\t@p add.s32 %1, %1, 1;\n\t"
          "@!p add.s32 %0, %0, 1;\n\t}"
          : "+r"(pos[q]), "+r"(pos[q2])
          : "d"(rem[q]), "d"(rem[q2]));
    }
  }
  int extra = L - assigned, ex_mod = extra;
  if (extra < 0 || extra >= S) {  // rare: more than one round of the round-robin
    const int ex_div = extra / S;
    ex_mod = extra % S;
#pragma unroll
    for (int q = 0; q < NS; ++q) lay[q] += ex_div;
  }
  bool zero = false;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    asm("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %1, %2;\n\t@p add.s32 %0, %0, 1;\n\t}"
        : "+r"(lay[q])
        : "r"(pos[q]), "r"(ex_mod));
    zero |= act[q] && lay[q] == 0;
  }
  if (zero) {  // every stage needs at least one layer (src/train_search.cpp:166-175)
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      if (act[q] && lay[q] == 0) {
        int dv = -1, dq = 0;
#pragma unroll
        for (int q2 = 0; q2 < NS; ++q2)
          if (act[q2] && lay[q2] > dv) {
            dv = lay[q2];
            dq = q2;
          }
#pragma unroll
        for (int q2 = 0; q2 < NS; ++q2)
          if (q2 == dq) lay[q2]--;
        lay[q] = 1;
      }
    }
  }
  // gather stage entries (train_cost_breakdown, src/cost_model.cpp:93-126). Totals and
  // computes are >= 0, infeasible entries hold +inf: plain ordered compares suffice.
  const double2* __restrict__ stage = tb.stage;
  double max_total = 0, max_comp = 0;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    if (act[q]) {
      const int b = q < NP ? vbi(q) : e.bi[q - NP];
      GP_CHECK(lay[q] >= 1 && lay[q] <= L && b >= 0);
      const double2 st = stage[(unsigned)(b * L + (lay[q] - 1))];
      asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %2, %0;\n\t@p mov.b64 %0, %2;\n\t"
          "setp.gt.f64 p, %3, %1;\n\t@p mov.b64 %1, %3;\n\t}"
          : "+d"(max_total), "+d"(max_comp)
          : "d"(st.x), "d"(st.y));
    }
  }
  if (DECODE) {
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      out_lay[q] = act[q] ? lay[q] : 0;
      out_bi[q] = act[q] ? (q < NP ? vbi(q) : e.bi[q - NP]) : -1;
    }
  }
  const bool feasible = max_total < __longlong_as_double(0x7ff0000000000000LL);
  if (!feasible) return false;
  // stage transfers in stage order: prefix-internal, junction, suffix-internal
  double transfers = D.transfers;
  if (R > 1) {
    const int e2 = sp.nc[R - 1] + 2;
    transfers += tb.tx[sp.tx_off[R > 1 ? R - 2 : 0] + (size_t)D.a_last * e2 + e.b1];
  }
#pragma unroll
  for (int j = 0; j < 3; ++j)
    if (j + 1 < k) transfers += e.t[j];
  const double fill = tb.fd_coef[S] * max_comp;
  per_step = max_total + fill + transfers;
  return true;
}


// ------------------------------------------- fast path: constant allocation total
// When every partial sum of the train set's device FLOPS is exact (all FLOPS are integer
// multiples of one power of two and their total stays below 2^53 of it — true for the
// spec-sheet FLOPS of every benchmark cluster, SURVEY.md 8a rule 2), allocate_layers'
// total is the same for every layout, so each block's share L*f/total, its floor and its
// remainder are per-block constants (K2e). A layout's layer counts then follow from the
// floors and from which stages the remainder ranking promotes by one, and both sides of
// a layout (prefix stages, suffix stages) can tabulate their stage maxima per promotion
// count (prefix: per warp, suffix: K2f). K1-fast merges the two sides with a rank count.
__global__ void k2e_block_shares(const double2* __restrict__ blkf, int nblk, double total,
                                 double2* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nblk) return;
  const double y = 1.0 / total;
  const double share = div_rn_recip(blkf[i].y, total, y);  // as eval_layout
  const int fl = static_cast<int>(share);
  out[i] = make_double2(share - fl, (double)fl);
}

constexpr int kFsBias = 1 << 20;  // suffix-stats encoding of the smallest floor sum

// K2m: one thread per choice of the middle run (R - 2): its MidRow — the k2f tables for a
// prefix side (promotion count a1 of its own stages, d1 water-filling donations taken from
// them; zero-layer stages counted with the one layer the fix-up gives them) — and its rank
// counts of the last run's blocks (#middle remainders >= x: prefix stages win ties).
__global__ void k2m_middle_rows(const SufEnt* __restrict__ mch, int n, const double2* __restrict__ blk_sh,
                                const double2* __restrict__ stage, int L, int blk_off_last, int nlast, int cw,
                                MidRow* __restrict__ rows, unsigned long long* __restrict__ cntb_mid) {
  constexpr int DM = kDonations;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const SufEnt e = mch[i];
  const int k = e.k;
  double rem[4];
  int fl[4], rk[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    rem[j] = -1.0;
    fl[j] = 0;
    if (j < k) {
      const double2 sh = blk_sh[e.bi[j]];
      rem[j] = sh.x;
      fl[j] = (int)sh.y;
    }
  }
  MidRow row;
  int fs = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    rk[j] = 0;
#pragma unroll
    for (int j2 = 0; j2 < 4; ++j2)
      if (j2 < k && j2 != j) rk[j] += rem[j2] > rem[j] || (rem[j2] == rem[j] && j2 < j);
    fs += fl[j];
    row.R[j] = -1.0;
  }
  for (int j = 0; j < k; ++j) row.R[rk[j]] = rem[j];
  for (int j = 0; j < 3; ++j) row.t[j] = e.t[j];
  row.k = (unsigned char)k;
  row.b1 = (unsigned char)e.b1;
  row.bl = (unsigned char)e.bl;
  row.fs = fs;
  unsigned bad = 0;
  for (int a = 0; a <= 4; ++a) {
    int lay[4];
    int nz = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      lay[j] = 0;
      if (j < k) {
        lay[j] = fl[j] + (rk[j] < a ? 1 : 0);
        nz += lay[j] == 0;
        if (lay[j] > L) bad |= 1u << a;
      }
    }
    row.nz[a] = (unsigned char)nz;
    bool live = true;
    for (int d = 0; d <= DM; ++d) {
      int mx = -1, jm = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < k && lay[j] > 0 && lay[j] > mx) {
          mx = lay[j];
          jm = j;
        }
      double mt = 0, mc = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= k) continue;
        const int l1 = lay[j] == 0 ? 1 : lay[j];
        if (l1 < 1 || l1 > L) continue;
        const double2 st = stage[(unsigned)(e.bi[j] * L + (l1 - 1))];
        if (st.x > mt) mt = st.x;
        if (st.y > mc) mc = st.y;
      }
      row.mp[a][d] = (signed char)(live ? (mx > 127 ? 127 : mx) : -1);
      row.pt[a][d] = make_double2(mt, mc);
      if (mx < 2) live = false;  // a donor needs >= 2 layers
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (live && j == jm) lay[j]--;
    }
  }
  row.bad = (int)bad;
  rows[i] = row;
  for (int w = 0; w < cw; ++w) {
    unsigned long long v = 0;
    for (int bq = 0; bq < 8; ++bq) {
      const int x = 8 * w + bq;
      if (x >= nlast) break;
      const double xr = blk_sh[blk_off_last + x].x;
      unsigned long long c = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) c += (j < k && row.R[j] >= xr) ? 1u : 0u;
      v |= c << (8 * bq);
    }
    cntb_mid[(size_t)i * cw + w] = v;
  }
}

// Per suffix choice: the fast-path tables (TrainTables::sf_*) and, per promotion count b and
// donation count d, the (max total, max compute) of its stages — zero-layer stages counted
// with the one layer the fix-up gives them, donors with the layers they keep.
constexpr long long kFastMinSuffixes = 32;  // K1-fast: least mean last-run choices per prefix
constexpr int kMaxLastBlocks = 256;  // per-warp rank-count bytes; the fast path takes <= 255 last-run blocks (else generic K1)
// suffix stage slots past k point at this rank-count entry, which holds kSentinelCount: its
// promotion test (count + j < extra) never holds, so the scan needs no per-suffix slot mask
constexpr int kSentinelBlock = 255;  // (byte ids: the fast path takes <= 255 last-run blocks)
constexpr unsigned kSentinelCount = 124;  // + j + 1 <= 128 for j <= 3: no borrow between bytes

__global__ void k2f_suffix_fast(const SufEnt* __restrict__ suf, int n, const double2* __restrict__ blk_sh,
                                const double2* __restrict__ stage, int L, int blk_off_last,
                                int4* __restrict__ sf_hot, double* __restrict__ sf_t,
                                signed char* __restrict__ sf_ms, double2* __restrict__ sf_st,
                                int* __restrict__ nzs_max) {
  constexpr int DM = kDonations;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const SufEnt e = suf[i];
  const int k = e.k;
  double rem[4];
  int fl[4], rk[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    rem[j] = -1.0;
    fl[j] = 0;
    if (j < k) {
      const double2 sh = blk_sh[e.bi[j]];
      rem[j] = sh.x;
      fl[j] = (int)sh.y;
    }
  }
  int fs = 0;
  int rbs[4] = {kSentinelBlock, kSentinelBlock, kSentinelBlock, kSentinelBlock};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    rk[j] = 0;
#pragma unroll
    for (int j2 = 0; j2 < 4; ++j2)
      if (j2 < k && j2 != j) rk[j] += rem[j2] > rem[j] || (rem[j2] == rem[j] && j2 < j);
    fs += fl[j];
  }
  for (int j = 0; j < k; ++j) rbs[rk[j]] = e.bi[j] - blk_off_last;
  reinterpret_cast<double2*>(sf_t)[i] = make_double2(e.t[0], e.t[1]);  // plane (t0, t1)[n]
  sf_t[2 * (size_t)n + i] = e.t[2];                                     // plane t2[n]
  unsigned nzs = 0, nz4 = 0, bad = 0;
  for (int b = 0; b <= 4; ++b) {
    int lay[4];
    int nz = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      lay[j] = 0;
      if (j < k) {
        lay[j] = fl[j] + (rk[j] < b ? 1 : 0);
        nz += lay[j] == 0;
        if (lay[j] > L) bad |= 1u << b;
      }
    }
    if (b < 4) nzs |= (unsigned)nz << (8 * b);
    else nz4 = (unsigned)nz;
    bool live = true;
    for (int d = 0; d <= DM; ++d) {
      int mx = -1, jm = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (j < k && lay[j] > 0 && lay[j] > mx) {
          mx = lay[j];
          jm = j;
        }
      double mt = 0, mc = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= k) continue;
        const int l1 = lay[j] == 0 ? 1 : lay[j];
        if (l1 < 1 || l1 > L) continue;
        const double2 st = stage[(unsigned)(e.bi[j] * L + (l1 - 1))];
        if (st.x > mt) mt = st.x;
        if (st.y > mc) mc = st.y;
      }
      sf_ms[(size_t)i * kMsStride + b * (DM + 1) + d] = (signed char)(live ? (mx > 127 ? 127 : mx) : -1);
      sf_st[(size_t)(b * (DM + 1) + d) * n + i] = make_double2(mt, mc);
      if (mx < 2) live = false;  // a donor needs >= 2 layers (checked by the scan)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (live && j == jm) lay[j]--;
    }
  }
  // (fs, nz4 | k << 8 | junction byte offset << 16, stage block ids in remainder order as bytes,
  // zero-layer counts at b = 0..3 as bytes): with nz4 as byte 4, byte b of {y:w} is one PRMT
  (void)bad;
  sf_hot[i] = make_int4(fs, (int)nz4 | (k << 8) | ((e.b1 * 8) << 16),
                        rbs[0] | (rbs[1] << 8) | (rbs[2] << 16) | (rbs[3] << 24), (int)nzs);
  int zmax = (int)nz4;
#pragma unroll
  for (int b = 0; b < 4; ++b) zmax = max(zmax, (int)((nzs >> (8 * b)) & 0xff));
  atomicMax(nzs_max, zmax);
  atomicMax(nzs_max + 1, kFsBias - fs);  // suffix floor-sum range: min via the bias
  atomicMax(nzs_max + 2, fs);
  // most zero-layer stages per (floor sum, promotion count): bounds the fix-ups a prefix
  // promotion count can meet (a candidate with promotions a, b has fs = L - fp - a - b)
  if (fs >= 0 && fs <= L)
    for (int b = 0; b <= 4; ++b) {
      const int z = b < 4 ? (int)((nzs >> (8 * b)) & 0xff) : (int)nz4;
      if (z > 0) atomicMax(nzs_max + 3 + fs * 5 + b, z);
    }
}

constexpr int kK1Threads = 128;
// K1-fast variant switches (A/B measurements with tools/build_variant.sh + k1_variants.sh);
// the defaults are the product
#ifndef GPV_CTAS
#define GPV_CTAS 6   // K1-fast launch bounds: min CTAs per SM (6: 72 registers, 7 resident; 7: same, 5: -17%)
#endif
#ifndef GPV_DYN
#define GPV_DYN 1    // K1-fast: prefix chunks handed out by an atomic counter (finer, balanced)
#endif
#ifndef GPV_GS
#define GPV_GS 4     // lanes per promotion count in the per-prefix tables
#endif
#ifndef GPV_ITEMS
#define GPV_ITEMS 24  // K1-fast: work items per warp (atomic-counter chunks; 12 and 48: -0.5 / -1 %)
#endif
#ifndef GPV_MINCHUNK
#define GPV_MINCHUNK 16  // K1-fast: least prefixes per work item (1.5e8-layout set: 1.07 -> 0.81 ms; 64: 0.92)
#endif
#ifndef GPV_UNROLL
#define GPV_UNROLL 2  // K1-fast candidate loop unroll
#endif
#define GPV_PRAGMA_(x) _Pragma(#x)
#define GPV_PRAGMA(x) GPV_PRAGMA_(x)
#ifndef GPV_MERGE
#define GPV_MERGE 1  // 1: zero-layer donors by the co-rank of the two donor sequences (no loop) (-0.4 ms)
#endif
constexpr int kZsTable = 128;  // > L on the fast path
// (the per-warp tables are kept small: the K1-fast CTAs' shared memory decides how much of the
// SM's 256 KB stays L1 for the suffix tables, which every candidate reads)

// Warp-uniform fast-path data of one prefix (shared memory): the tables the candidate loop
// reads (pt, mp, nzp, fp, bad) and, for R >= 3, the FRONT runs' own tables (runs 0..R-3,
// rebuilt only when the front combination changes), which the per-prefix merge combines
// with the middle run's precomputed row (MidRow).
template <int R>
struct PrefixFast {
  static constexpr int NP = (R - 1) * kMaxPerRun;
  static constexpr int NPF = (R > 2 ? R - 2 : 0) * kMaxPerRun;  // front slots
  static constexpr int NQF = NPF > 0 ? NPF : 1;
  static constexpr int NPFP = NPF < 4 ? 4 : (NPF < 8 ? 8 : 16);  // > NPF, power of two
  static constexpr int DM = kDonations;
  // merged prefix tables (what the candidate loop reads)
  double2 pt[NP + 1][DM + 1]; // (max total, max compute) of the prefix stages: top a promoted, d donations
  short mp[NP + 1][DM + 1];   // largest layer count after d donations (-1: none / invalid)
  unsigned char nzp[NP + 1];  // zero-layer prefix stages at promotion a
  int fp;                     // sum of the prefix floors
  int bad;                    // bit a: a promoted prefix stage would exceed L layers
  // front tables (runs 0..R-3)
  double srtf[NPFP];          // front remainders sorted (desc, stage order), padded with -1
  double2 tcf[NQF][DM + 3];   // front stage q's (total, compute) at fl+1-o layers, o = DM+2: 1 layer
  double remf[NQF];
  int flf[NQF];
  int rkf[NQF];
  int bif[NQF];
  double termf[NQF];          // per front slot: the stage-transfer term that follows it (0 if none)
  bool actf[NQF];
  double2 ptf[NPF + 1][DM + 1];
  short mpf[NPF + 1][DM + 1];
  unsigned char nzf[NPF + 1];
  int kf, fpf, badf, a_lastf; // front stages, floor sum, over bits, start of the front's last block
  double trf;                 // left fold of the front's stage transfers
  long long fkey;             // front combination the front tables hold (-1: none)
  MidRow mrow[2];             // the middle rows of this prefix and (prefetched by cp.async) the next
  int mrow_c[2];              // middle choice held by each buffer (-1: none)
  int mbuf;                   // buffer of the current prefix
  int cnt1[NPFP];             // per sorted front entry: middle remainders strictly above it

#ifdef GP_DEBUG_CHECKS
  int a_lo, a_hi;             // the tabulated promotion counts
  int dm[NP + 1];             // the tabulated donations per promotion count
#endif
};

// K1-fast shared memory per warp beside PrefixFast: the rank count of every last-run
// block's remainder among the prefix's (cntb) and the prefix's junction-transfer row (txs).
constexpr int kMaxJunction = 32;  // nc_last + 2 (else generic K1)
struct __align__(8) PrefixLast {
  unsigned char cntb[kMaxLastBlocks];      // rank counts among all prefix remainders (merged); [255]: sentinel
  unsigned char cntbf[kMaxLastBlocks];     // among the front's remainders only (rebuilt with the front)
  double txs[kMaxJunction];
  double fdk[8];                           // fill/drain coefficient of S = (prefix stages) + k stages
};

// number of entries >= x in the descending, -1-padded srt (x >= 0)
template <int R>
__device__ __forceinline__ int count_ge(const double* srt, double x) {
  constexpr int NPP = PrefixFast<R>::NPFP;
  int pos = 0;
#pragma unroll
  for (int step = NPP / 2; step >= 1; step >>= 1)
    if (srt[pos + step - 1] >= x) pos += step;
  return pos;
}

// 16-byte asynchronous global -> shared copies (LDGSTS): the next prefix's middle row is
// fetched while the current prefix's candidates are scored.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// All lanes: start copying middle row c into buffer b (one 16-byte chunk per lane)
template <int R>
__device__ __forceinline__ void mid_fetch(int lane, const TrainTables& tb, PrefixFast<R>& F, int b, int c) {
  static_assert(sizeof(MidRow) == 32 * 16, "one 16-byte chunk per lane");
  const char* src = reinterpret_cast<const char*>(tb.mid + c);
  char* dst = reinterpret_cast<char*>(&F.mrow[b]);
  cp_async16(dst + 16 * lane, src + 16 * lane);
  cp_async_commit();
  if (lane == 0) F.mrow_c[b] = c;
}

// K1-fast's prefix step (lane 0): the tables need only the middle run's choice index, the
// prefix stage count (kf + the middle row's k) and the rank base, so while the middle run has
// a next choice within the stage budget only those advance; the middle run's cut positions
// and P.u are left stale. At the middle run's last choice they are restored and the full
// odometer (prefix_advance) carries into the front runs and resets the middle run.
template <int R>
__device__ __forceinline__ void prefix_advance_fast(const TrainSpace& sp, Prefix<R>& P, int u_cur) {
  if constexpr (R < 2) {
    prefix_advance<R>(sp, P);
  } else {
    constexpr int rm = R - 2;
    int used = 0;
#pragma unroll
    for (int r = 0; r < rm; ++r) used += P.k[r];
    const int nc = sp.nc[rm];
    // the middle run's largest stage count the odometer reaches (prefix_advance's growth test)
    const int kallow = min(min(sp.kmax[rm], sp.max_stages - used - 1), nc + 1);
    long long nallow = 0;  // its choices with 1..kallow stages (run_compositions order)
#pragma unroll
    for (int k = 1; k <= kMaxPerRun; ++k)
      if (k <= kallow) nallow += binom_small(nc, k - 1);
    if (P.ci[rm] + 1 < nallow) {
      P.base += sp.cnt[R - 1][u_cur];
      P.ci[rm]++;
      return;
    }
    const int m = kallow - 1;  // the last choice: cut positions nc - m + 1 .. nc
    P.k[rm] = kallow;
    P.b[rm][0] = 0;
#pragma unroll
    for (int j = 1; j <= kMaxPerRun; ++j) {
      if (j <= m) P.b[rm][j] = nc - (m - j);
      else if (j == m + 1) P.b[rm][j] = nc + 1;
    }
    P.u = used + kallow;
    GP_CHECK(P.u == u_cur);
    prefix_advance<R>(sp, P);
  }
}

// R == 1 (no prefix runs): empty prefix tables.
template <int R>
__device__ __forceinline__ void prefix_single(int lane, PrefixData<R>& D, PrefixFast<R>& F, unsigned char* cntb,
                                              int nlast) {
  constexpr int DM = kDonations;
  if (lane <= DM) {
    F.pt[0][lane] = make_double2(0.0, 0.0);
    F.mp[0][lane] = -1;
  }
  if (lane == 0) {
    F.fp = 0;
    F.bad = 0;
    F.nzp[0] = 0;
    D.transfers = 0.0;
    D.a_last = 0;
    D.u = 0;
  }
  for (int i = lane; i < nlast; i += 32) cntb[i] = 0;
  __syncwarp();
}

// All lanes: the front runs' (0..R-3) tables — slot data, remainder ranks, stage-time cache,
// the full (promotion a0 in [0, kf], donation d0 <= kDonations) tables, the front transfer
// fold and the rank counts of the last run's blocks among the front remainders. Rebuilt only
// when the front combination changes (every ~#middle-choices prefixes).
template <int R>
__device__ __forceinline__ void front_fast(int lane, const TrainSpace& sp, const TrainTables& tb, int L,
                                           const Prefix<R>& P, PrefixFast<R>& F, unsigned char* cntbf, int nlast) {
  constexpr int NPF = PrefixFast<R>::NPF;
  constexpr int NPFP = PrefixFast<R>::NPFP;
  constexpr int DM = kDonations;
  if (NPF == 0) {  // R == 2: no front
    if (lane <= DM) {
      F.ptf[0][lane] = make_double2(0.0, 0.0);
      F.mpf[0][lane] = -1;
    }
    if (lane < NPFP) F.srtf[lane] = -1.0;
    if (lane == 0) {
      F.nzf[0] = 0;
      F.kf = F.fpf = F.badf = F.a_lastf = 0;
      F.trf = 0.0;
    }
    for (int i = lane; i < nlast; i += 32) cntbf[i] = 0;
    __syncwarp();
    return;
  }
  bool aq = false;
  double rq = -1.0;
  int fq = 0;
  if (lane < NPF) {
    const int r = lane / kMaxPerRun, j = lane % kMaxPerRun;
    const bool act = j < P.k[r];
    int bi = 0;
    double t = 0.0;
    if (act) {
      bi = sp.blk_off[r] + blk_index(sp.nc[r], P.b[r][j], P.b[r][j + 1]);
      if (j + 1 < P.k[r]) {
        const int e = sp.nc[r] + 2;
        t = tb.tin[sp.tin_off[r] + ((size_t)P.b[r][j] * e + P.b[r][j + 1]) * e +
                   P.b[r][j + 2 <= kMaxPerRun ? j + 2 : kMaxPerRun]];
      } else if (r + 3 < R) {  // junction to the next front run
        const int e2 = sp.nc[r + 1] + 2;
        t = tb.tx[sp.tx_off[r] + (size_t)P.b[r][j] * e2 + P.b[r + 2 < R ? r + 1 : r][1]];
      } else {  // the front's last block: its junction to the middle run is per prefix
        F.a_lastf = P.b[r][j];
      }
      const double2 sh = tb.blk_sh[bi];
      rq = sh.x;
      fq = (int)sh.y;
    }
    aq = act;
    F.actf[lane] = act;
    F.bif[lane] = bi;
    F.termf[lane] = t;
    F.remf[lane] = rq;
    F.flf[lane] = fq;
  }
  if (lane < NPFP) F.srtf[lane] = -1.0;
  if (lane == 0) F.badf = 0;
  __syncwarp();
  if (lane < NPF && aq) {
    int rk = 0;
#pragma unroll
    for (int q2 = 0; q2 < NPF; ++q2) {
      const double r2 = F.remf[q2];
      rk += (F.actf[q2] && (r2 > rq || (r2 == rq && q2 < lane))) ? 1 : 0;
    }
    F.rkf[lane] = rk;
    F.srtf[rk] = rq;
  }
  for (int idx = lane; idx < NPF * (DM + 3); idx += 32) {
    const int q = idx / (DM + 3), o = idx % (DM + 3);
    if (!F.actf[q]) continue;
    const int lay = o == DM + 2 ? 1 : F.flf[q] + 1 - o;
    double2 v = make_double2(kInf, kInf);
    if (lay >= 1 && lay <= L) v = tb.stage[(unsigned)(F.bif[q] * L + (lay - 1))];
    F.tcf[q][o] = v;
  }
  __syncwarp();
  int kf = 0;
#pragma unroll
  for (int r = 0; r + 2 < R; ++r) kf += P.k[r];
  // One group of GS lanes per promotion count a0 in [0, kf], up to kDonations water-filling
  // donations each (the first slot with the most layers donates).
  constexpr int GS = GPV_GS;
  constexpr int SPL = NPF > 0 ? (NPF + GS - 1) / GS : 1;
  constexpr int GPW = 32 / GS;
  const int grp = lane / GS, ql = lane % GS;
  bool actv[SPL];
  int flv[SPL], rkv[SPL];
#pragma unroll
  for (int j = 0; j < SPL; ++j) {
    const int q = ql + GS * j;
    actv[j] = q < NPF && F.actf[q];
    flv[j] = actv[j] ? F.flf[q] : 0;
    rkv[j] = actv[j] ? F.rkf[q] : 0;
  }
  const unsigned gmask = ((1u << GS) - 1u) << (grp * GS);
  for (int a0 = 0; a0 <= kf; a0 += GPW) {
    const int a = a0 + grp;
    const bool ga = a <= kf;
    int lay[SPL];
    int nz = 0;
    bool ov = false;
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
      lay[j] = actv[j] ? flv[j] + (rkv[j] < a ? 1 : 0) : 0;
      nz += (actv[j] && lay[j] == 0) ? 1 : 0;
      ov |= actv[j] && lay[j] > L;
    }
#pragma unroll
    for (int o = GS / 2; o >= 1; o >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, o);
    const bool over = (__ballot_sync(0xffffffffu, ov) & gmask) != 0;
    bool live = true;
    for (int d = 0; d <= DM; ++d) {
      double vx = 0, vy = 0;  // an inactive slot adds nothing (the maxima start at 0)
      int key = -1;           // most layers, then the first slot
#pragma unroll
      for (int j = 0; j < SPL; ++j) {
        if (!actv[j]) continue;
        const int q = ql + GS * j;
        const double2 v = F.tcf[q][lay[j] == 0 ? DM + 2 : flv[j] + 1 - lay[j]];
        const double tx = v.x > 0 ? v.x : 0.0, ty = v.y > 0 ? v.y : 0.0;
        if (tx > vx) vx = tx;
        if (ty > vy) vy = ty;
        if (lay[j] > 0) key = max(key, lay[j] * 16 + (15 - q));
      }
#pragma unroll
      for (int o = GS / 2; o >= 1; o >>= 1) {
        const double ox = __shfl_xor_sync(0xffffffffu, vx, o), oy = __shfl_xor_sync(0xffffffffu, vy, o);
        const int ok = __shfl_xor_sync(0xffffffffu, key, o);
        if (ox > vx) vx = ox;
        if (oy > vy) vy = oy;
        key = max(key, ok);
      }
      const int mx = key < 0 ? -1 : key >> 4;
      const int qm = key < 0 ? -1 : 15 - (key & 15);
      if (ga && ql == 0) {
        F.ptf[a][d] = make_double2(vx, vy);
        F.mpf[a][d] = (short)(live ? mx : -1);
      }
      if (mx < 2) live = false;
      if (live) {
#pragma unroll
        for (int j = 0; j < SPL; ++j)
          if (actv[j] && ql + GS * j == qm) --lay[j];
      }
    }
    if (ga && ql == 0) {
      F.nzf[a] = (unsigned char)nz;
      if (over) atomicOr(&F.badf, 1 << a);
    }
  }
  if (lane == 0) {
    int fp = 0;
    double tr = 0.0;
#pragma unroll
    for (int q = 0; q < NPF; ++q) {
      fp += F.flf[q];  // inactive slots hold 0
      tr += F.termf[q];
    }
    F.kf = kf;
    F.fpf = fp;
    F.trf = tr;
  }
  for (int i = lane; i < nlast; i += 32)
    cntbf[i] = (unsigned char)count_ge<R>(F.srtf, tb.blk_sh[sp.blk_off[R - 1] + i].x);
  __syncwarp();
}

// All lanes: the prefix tables of (front combination, middle choice) — the merge of the
// front tables and the middle run's MidRow. Promotions: the prefix's top-a stages by
// remainder (ties: the earlier stage, i.e. the front) hold a0 front and a1 = a - a0 middle
// stages; donations: the first stage with the most layers donates, so the d donors are the
// d largest of the two non-increasing donor sequences (front first on ties, co-rank); the
// maxima of a state are the maxima of the two sides' states. Then the transfer fold (front,
// junction into the middle run, its internal terms), the merged rank counts and the
// junction row to the last run.
template <int R>
__device__ __forceinline__ void prefix_merge(int lane, const TrainSpace& sp, const TrainTables& tb, int L,
                                             int3 sstat, const Prefix<R>& P, PrefixData<R>& D, PrefixFast<R>& F,
                                             PrefixLast& PL, const unsigned char* zst, int nlast) {
  constexpr int NPF = PrefixFast<R>::NPF;
  constexpr int DM = kDonations;
  const int c1 = P.ci[R - 2];
  // this prefix's middle row: normally prefetched into the other buffer during the previous
  // prefix; else (chunk start, a front change) fetched now
  int b = F.mbuf ^ 1;
  if (F.mrow_c[b] != c1) {
    b = F.mbuf;  // (the current buffer's row is no longer needed)
    mid_fetch<R>(lane, tb, F, b, c1);
  }
  cp_async_wait_all();
  __syncwarp();
  if (lane == 0) F.mbuf = b;
  const MidRow& M = F.mrow[b];
  const int kf = F.kf, k1 = M.k;
  if (lane < NPF) {
    int c = 0;
    const double rf = F.srtf[lane];
#pragma unroll
    for (int j = 0; j < 4; ++j) c += (j < k1 && M.R[j] > rf) ? 1 : 0;
    F.cnt1[lane] = c;
  }
  if (lane == 0) {
    F.bad = 0;
    D.u = kf + k1;  // (P.u is not maintained by prefix_advance_fast)
  }
  __syncwarp();
  const int fp_all = F.fpf + M.fs;
  const int kp = kf + k1;
  const int nzs_max = sstat.x, fs_min = kFsBias - sstat.y, fs_max = sstat.z;
  const int a_lo = max(0, L - fp_all - fs_max - 4), a_hi = min(kp, L - fp_all - fs_min);
#ifdef GP_DEBUG_CHECKS
  if (lane == 0) {
    F.a_lo = a_lo;
    F.a_hi = a_hi;
  }
#endif
  const int ncell = a_hi >= a_lo ? (a_hi - a_lo + 1) * (DM + 1) : 0;
  // a0(a) = #{front entries i < kf : i + cnt1[i] < a}, the keys held in registers (the cell
  // loop's shared-memory stores would otherwise force a reload per cell)
  int key[NPF > 0 ? NPF : 1];
#pragma unroll
  for (int i = 0; i < NPF; ++i) key[i] = i < kf ? i + F.cnt1[i] : (1 << 20);
  for (int idx = lane; idx < ncell; idx += 32) {
    const int a = a_lo + idx / (DM + 1), d = idx % (DM + 1);
    int a0 = 0;
#pragma unroll
    for (int i = 0; i < NPF; ++i) a0 += key[i] < a ? 1 : 0;
    const int a1 = a - a0;
    GP_CHECK(a1 >= 0 && a1 <= k1 && a0 <= kf);
    const int nz = F.nzf[a0] + M.nz[a1];
    const int za = fp_all + a;
    const int zs = za < kZsTable ? zst[za] : 0;
    const int dm = min(DM, nz + min(zs, nzs_max));
    if (d == 0) {
      F.nzp[a] = (unsigned char)nz;
#ifdef GP_DEBUG_CHECKS
      if (((F.badf >> a0) | (M.bad >> a1)) & 1) atomicOr(&F.bad, 1 << a);
      F.dm[a] = dm;
#endif
    }
    if (d > dm) continue;
    int d0 = 0;
    if (d > 0) {  // common cases first: every donor from one side
      if (F.mpf[a0][d - 1] >= M.mp[a1][0]) {
        d0 = d;
      } else if (M.mp[a1][d - 1] > F.mpf[a0][0]) {
        d0 = 0;
      } else {
#pragma unroll
        for (int i = 1; i <= DM; ++i)
          if (i <= d) d0 += F.mpf[a0][i - 1] >= M.mp[a1][d - i] ? 1 : 0;
      }
    }
    const int d1 = d - d0;
    const double2 pf = F.ptf[a0][d0], pm = M.pt[a1][d1];
    double2 v = pf;
    if (pm.x > v.x) v.x = pm.x;
    if (pm.y > v.y) v.y = pm.y;
    bool live = true;
    if (d > 0) {  // the donors so far: the smallest (last) one must have had >= 2 layers
      const int lf = d0 > 0 ? F.mpf[a0][d0 - 1] : 0x7fff, lm = d1 > 0 ? M.mp[a1][d1 - 1] : 0x7fff;
      live = (lf < lm ? lf : lm) >= 2;
    }
    const int mxf = F.mpf[a0][d0], mxm = M.mp[a1][d1];
    F.pt[a][d] = v;
    F.mp[a][d] = (short)(live ? (mxf > mxm ? mxf : mxm) : -1);
  }
  if (lane == 0) {
    F.fp = fp_all;
    double tr = F.trf;
    if (R > 2) tr += tb.tx[sp.tx_off[R > 2 ? R - 3 : 0] + (size_t)F.a_lastf * (sp.nc[R - 2] + 2) + M.b1];
    tr += M.t[0];  // (absent internal terms are exact zeros)
    tr += M.t[1];
    tr += M.t[2];
    D.transfers = tr;
    D.a_last = M.bl;
  }
  {
    const int cw = tb.cw;
    unsigned long long* __restrict__ dst = reinterpret_cast<unsigned long long*>(PL.cntb);
    const unsigned long long* srcf = reinterpret_cast<const unsigned long long*>(PL.cntbf);
    const unsigned long long* __restrict__ srcm = tb.cntb_mid + (size_t)c1 * cw;
    for (int w = lane; w < cw; w += 32) dst[w] = srcf[w] + __ldg(srcm + w);  // bytes < 128: no carries
  }
  __syncwarp();
  const int e2 = sp.nc[R - 1] + 2;
  const double* __restrict__ txrow = tb.tx + sp.tx_off[R > 1 ? R - 2 : 0] + (size_t)D.a_last * e2;
  for (int i = lane; i < e2; i += 32) PL.txs[i] = txrow[i];
  // prefetch the next prefix's middle row (usually the next middle choice)
  if (c1 + 1 < tb.n_mid) mid_fetch<R>(lane, tb, F, b ^ 1, c1 + 1);
  __syncwarp();
}

struct ScanRange {
  long long p_lo, s_lo, p_hi, s_hi;  // candidates (p, s) with (p_lo,s_lo) <= (p,s) < (p_hi,s_hi)
  long long n_pref;                  // prefixes touched
  long long chunk;                   // prefixes per warp work item
  int defer_all;                     // test hook (GPLAN_K1_DEFER_ALL=1): K1-fast defers every candidate
  unsigned long long* work;          // K1-fast: next work item (zeroed per launch)
  double* dump;                      // test hook (DUMP instantiations): per_step of rank r in
  long long dump_lo, dump_hi;        //   [dump_lo, dump_hi) at dump[r - dump_lo]
};

constexpr int kDeferBlocks = 64;  // CTAs of k1_deferred (their partials follow K1-fast's)

__device__ __forceinline__ NearMin nm_shfl_xor(const NearMin& m, int o) {
  NearMin r;
  r.b0 = __shfl_xor_sync(0xffffffffu, m.b0, o);
#pragma unroll
  for (int i = 0; i < 3; ++i) r.key[i] = __shfl_xor_sync(0xffffffffu, m.key[i], o);
  r.feasible = __shfl_xor_sync(0xffffffffu, m.feasible, o);
  return r;
}

// CTA-wide merge of a CTA of at most NW warps; the result is valid in thread 0.
template <int NW = 32>
__device__ NearMin nm_block_reduce(NearMin m) {
  __shared__ NearMin sb[NW];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nm_merge(m, nm_shfl_xor(m, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sb[wid] = m;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    if (lane < nw) {
      m = sb[lane];
    } else {
      nm_init(m);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nm_merge(m, nm_shfl_xor(m, o));
  }
  return m;
}

// The generic scan of work items warp, warp + n_warps, ... (prefix chunks) of a range;
// returns the thread's summary. P/D: the warp's shared-memory prefix state.
template <int R, bool DUMP = false>
__device__ __forceinline__ NearMin k1_scan_warps(const TrainSpace& sp, const TrainTables& tb,
                                                 const double2* __restrict__ blkf, int L, const ScanRange& rg,
                                                 long long warp, long long n_warps, Prefix<R>& P,
                                                 PrefixData<R>& D) {
  const int lane = threadIdx.x & 31;
  const long long n_items = (rg.n_pref + rg.chunk - 1) / rg.chunk;
  // thread summary in registers: NearMin {b0, k0..k2, feasible}
  long long b0 = kInfBits, k0 = LLONG_MAX, k1 = LLONG_MAX, k2 = LLONG_MAX, feasible = 0;
  for (long long it = warp; it < n_items; it += n_warps) {
    long long p = rg.p_lo + it * rg.chunk;
    const long long p_end = min(p + rg.chunk, rg.p_lo + rg.n_pref);
    __syncwarp();
    if (lane == 0) prefix_decode<R>(sp, p, P);
    for (; p < p_end; ++p) {
      __syncwarp();
      if (lane == 0) prefix_data<R>(sp, tb, blkf, P, D);
      __syncwarp();
      const long long ns = sp.cnt[R - 1][D.u];
      const long long s0 = p == rg.p_lo ? rg.s_lo : 0;
      const long long s1 = p == rg.p_hi ? rg.s_hi : ns;
      const long long pbase = P.base;  // keys are ranks: base of the prefix + suffix index
      for (long long s = s0 + lane; s < s1; s += 32) {
        const SufEnt e = tb.suf[s];
        double x;
        const bool ok = eval_layout<R, false>(sp, tb, blkf, L, D, e, x, nullptr, nullptr);
        if (DUMP && pbase + s >= rg.dump_lo && pbase + s < rg.dump_hi)
          rg.dump[pbase + s - rg.dump_lo] = ok ? x : __longlong_as_double(0x7ff0000000000000LL);
        if (ok) {
          ++feasible;
          // keys grow along a thread's walk: only a new minimum or a pattern within two
          // ulps of it can change the summary, and a pattern already held keeps its key
          const long long d = __double_as_longlong(x) - b0;
          if (d < 3) {
            const long long key = pbase + s;
            if (d < 0) {  // new minimum: shift the held patterns up by -d
              k2 = d == -1 ? k1 : d == -2 ? k0 : LLONG_MAX;
              k1 = d == -1 ? k0 : LLONG_MAX;
              k0 = key;
              b0 += d;
            } else if (d == 1) {
              k1 = min(k1, key);
            } else if (d == 2) {
              k2 = min(k2, key);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0 && p + 1 < p_end) prefix_advance<R>(sp, P);
    }
  }
  return NearMin{b0, {k0, k1, k2}, feasible};
}

template <int R, bool DUMP = false>
__global__ void __launch_bounds__(kK1Threads, R <= 3 ? 4 : 2) k1_layout_scan(TrainSpace sp, TrainTables tb,
                                                      const double2* __restrict__ blkf, int L,
                                                      ScanRange rg, NearMin* __restrict__ partial) {
  // the warp's current prefix lives in shared memory (lane 0 owns it; lanes read broadcasts)
  __shared__ Prefix<R> sP[kK1Threads / 32];
  __shared__ PrefixData<R> sD[kK1Threads / 32];
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
  NearMin nm = k1_scan_warps<R, DUMP>(sp, tb, blkf, L, rg, warp, n_warps, sP[threadIdx.x >> 5], sD[threadIdx.x >> 5]);
  nm = nm_block_reduce(nm);
  if (threadIdx.x == 0) partial[blockIdx.x] = nm;
}

// The generic scan for spaces whose last type run has few choices (a last run of one or two
// machines: a handful of suffixes per prefix, so a warp per prefix would leave most lanes idle
// and pay the serial prefix tabulation per handful of candidates). Each warp splits into
// G = 32 / GS groups of GS lanes; group g walks the g-th contiguous slice of the warp's chunk
// (one decode, then the odometer), the G groups in lockstep — their leaders tabulate G
// prefixes at once — and each group's lanes the prefix's suffixes. A thread's keys grow along
// its walk.
template <int R, int GS, bool DUMP = false>
__global__ void __launch_bounds__(kK1Threads, R <= 3 ? 4 : 2) k1_layout_scan_grouped(TrainSpace sp, TrainTables tb,
                                                      const double2* __restrict__ blkf, int L,
                                                      ScanRange rg, NearMin* __restrict__ partial) {
  constexpr int G = 32 / GS;
  // groups share their prefix through shared memory; with one lane per prefix (GS == 1) the
  // lane keeps it in its own (local) memory: per-lane structs in shared memory would put every
  // lane's same field in the same bank
  constexpr int GSH = GS == 1 ? 1 : G;
  __shared__ Prefix<R> sP[kK1Threads / 32][GSH];
  __shared__ PrefixData<R> sD[kK1Threads / 32][GSH];
  const int lane = threadIdx.x & 31, g = lane / GS, gl = lane % GS;
  Prefix<R> Pl;
  PrefixData<R> Dl;
  Prefix<R>& P = GS == 1 ? Pl : sP[threadIdx.x >> 5][GS == 1 ? 0 : g];
  PrefixData<R>& D = GS == 1 ? Dl : sD[threadIdx.x >> 5][GS == 1 ? 0 : g];
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long n_items = (rg.n_pref + rg.chunk - 1) / rg.chunk;
  long long b0 = kInfBits, k0 = LLONG_MAX, k1 = LLONG_MAX, k2 = LLONG_MAX, feasible = 0;
  for (long long it = warp; it < n_items; it += n_warps) {
    // group g walks its own contiguous slice of the work item: one decode, then the odometer
    const long long p0 = rg.p_lo + it * rg.chunk;
    const long long p_end = min(p0 + rg.chunk, rg.p_lo + rg.n_pref);
    const long long cl = (rg.chunk + G - 1) / G;
    long long p = p0 + g * cl;
    const long long q_end = min(p + cl, p_end);
    __syncwarp();
    if (gl == 0 && p < q_end) prefix_decode<R>(sp, p, P);
    for (long long t = 0; t < cl; ++t, ++p) {
      const bool has = p < q_end;
      __syncwarp();
      if (gl == 0 && has) prefix_data<R>(sp, tb, blkf, P, D);
      __syncwarp();
      long long s0 = 0, s1 = 0, pbase = 0;
      if (has) {
        const long long ns = sp.cnt[R - 1][D.u];
        s0 = p == rg.p_lo ? rg.s_lo : 0;
        s1 = p == rg.p_hi ? rg.s_hi : ns;
        pbase = P.base;
      }
      for (long long s = s0 + gl; s < s1; s += GS) {
        const SufEnt e = tb.suf[s];
        double x;
        const bool ok = eval_layout<R, false>(sp, tb, blkf, L, D, e, x, nullptr, nullptr);
        if (DUMP && pbase + s >= rg.dump_lo && pbase + s < rg.dump_hi)
          rg.dump[pbase + s - rg.dump_lo] = ok ? x : __longlong_as_double(0x7ff0000000000000LL);
        if (ok) {
          ++feasible;
          const long long d = __double_as_longlong(x) - b0;
          if (d < 3) {
            const long long key = pbase + s;
            if (d < 0) {
              k2 = d == -1 ? k1 : d == -2 ? k0 : LLONG_MAX;
              k1 = d == -1 ? k0 : LLONG_MAX;
              k0 = key;
              b0 += d;
            } else if (d == 1) {
              k1 = min(k1, key);
            } else if (d == 2) {
              k2 = min(k2, key);
            }
          }
        }
      }
      __syncwarp();
      if (gl == 0 && p + 1 < q_end) prefix_advance<R>(sp, P);
    }
  }
  NearMin nm{b0, {k0, k1, k2}, feasible};
  nm = nm_block_reduce(nm);
  if (threadIdx.x == 0) partial[blockIdx.x] = nm;
}

// candidates scored by K1-fast's tables / by the deferred generic kernel (GPLAN_PROFILE report)
__device__ unsigned long long g_k1_fast_cnt[2];

// K1-fast (constant allocation total). Keys are ranks (prefix base + suffix index), in
// increasing order along a thread's walk. Per candidate: the suffix's remainder ranks among
// the prefix's (cntb) fix how many prefix (a) and suffix (b) stages the round-robin
// promotes; zero-layer fix-ups are merged from the two sides' donation tables; the stage
// maxima are then two table reads. Layouts outside the tabulated cases (extra layers
// outside [0, S), more than kDonations fix-ups, a donor left without layers) are queued
// for k1_deferred, which scores them with the generic eval_layout — so every candidate's
// per-step time is the one the reference computes.
template <int R, bool DUMP = false>
__global__ void __launch_bounds__(kK1Threads, GPV_CTAS) k1_layout_scan_fast(TrainSpace sp, TrainTables tb,
                                                      const double2* __restrict__ blkf, int L,
                                                      ScanRange rg, NearMin* __restrict__ partial,
                                                      unsigned long long* __restrict__ slow_q) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long n_items = (rg.n_pref + rg.chunk - 1) / rg.chunk;
  const int nsuf32 = sp.n_suf;
  long long b0 = kInfBits, k0 = LLONG_MAX, k1 = LLONG_MAX, k2 = LLONG_MAX, feasible = 0;
  double xthr = __longlong_as_double(kInfBits);  // per-step times above bits b0 + 2 cannot matter
  unsigned n_tab = 0;
  __shared__ Prefix<R> sP[kK1Threads / 32];
  __shared__ PrefixData<R> sD[kK1Threads / 32];
  __shared__ PrefixFast<R> sF[kK1Threads / 32];
  Prefix<R>& P = sP[threadIdx.x >> 5];
  PrefixData<R>& D = sD[threadIdx.x >> 5];
  PrefixFast<R>& F = sF[threadIdx.x >> 5];
  const int e2 = sp.nc[R - 1] + 2;
  const int3 sstat = make_int3(tb.nzs_max[0], tb.nzs_max[1], tb.nzs_max[2]);
  __shared__ PrefixLast sL[kK1Threads / 32];
  __shared__ double fd[GP_MAX_STAGES + 1];
  unsigned char* const cntb = sL[threadIdx.x >> 5].cntb;
  double* const txs = sL[threadIdx.x >> 5].txs;
  for (int i = threadIdx.x; i <= GP_MAX_STAGES; i += blockDim.x) fd[i] = tb.fd_coef[i];
  // zst[t]: most zero-layer suffix stages over the (floor sum, promotion count b) pairs a
  // candidate whose prefix floors plus promotions total t can meet (fs = L - t - b)
  __shared__ unsigned char zst[kZsTable];
  for (int t = threadIdx.x; t < kZsTable; t += blockDim.x) {
    int z = 0;
    for (int b = 0; b <= 4; ++b) {
      const int fs = L - t - b;
      if (fs >= 0 && fs <= L) z = max(z, tb.nzs_max[3 + fs * 5 + b]);
    }
    zst[t] = (unsigned char)min(z, 255);
  }
  const int nlast = e2 * (e2 - 1) / 2;
  const int Lx = rg.defer_all ? -(1 << 20) : L;  // the test hook defers every candidate
  double* const fdk = sL[threadIdx.x >> 5].fdk;
  if ((threadIdx.x & 31) == 0) {
    // (per-prefix writes stop below the sentinel, or, with 249..255 blocks, add the middle
    // row's zero padding byte to the front's sentinel)
    cntb[kSentinelBlock] = (unsigned char)kSentinelCount;
    sL[threadIdx.x >> 5].cntbf[kSentinelBlock] = (unsigned char)kSentinelCount;
    F.fkey = -1;
    F.mrow_c[0] = F.mrow_c[1] = -1;
    F.mbuf = 0;
  }
  __syncthreads();
  #if GPV_DYN
  // the first item of each warp by its index, the next ones from the shared counter
  for (long long it = warp; it < n_items;) {
#else
  for (long long it = warp; it < n_items; it += n_warps) {
#endif
    long long p = rg.p_lo + it * rg.chunk;
    const long long p_end = min(p + rg.chunk, rg.p_lo + rg.n_pref);
    __syncwarp();
    if (lane == 0) prefix_decode<R>(sp, p, P);
    for (; p < p_end; ++p) {
      __syncwarp();
      if constexpr (R == 1) {
        prefix_single<R>(lane, D, F, cntb, nlast);
      } else {
        // the front runs' tables only when the front combination changed
        long long fk = 0;
#pragma unroll
        for (int r = 0; r + 2 < R; ++r) fk = (fk << 21) | P.ci[r];
        if (fk != F.fkey) {
          front_fast<R>(lane, sp, tb, L, P, F, sL[threadIdx.x >> 5].cntbf, nlast);
          if (lane == 0) F.fkey = fk;
        }
        prefix_merge<R>(lane, sp, tb, L, sstat, P, D, F, sL[threadIdx.x >> 5], zst, nlast);
      }
      const int kp = D.u;
      if (lane < 8) fdk[lane] = fd[min(kp + lane, GP_MAX_STAGES)];
      __syncwarp();
      const int fp = F.fp, pbad = F.bad;
      (void)pbad;  // (read by the debug checks)
      const double dtr = D.transfers;
      const long long ns = sp.cnt[R - 1][kp];
      const long long pbase = P.base;  // keys are ranks: base of the prefix + suffix index
      const long long s0 = p == rg.p_lo ? rg.s_lo : 0;
      const long long s1 = p == rg.p_hi ? rg.s_hi : ns;
      // table-scored count: every candidate of this lane, less the deferred ones (below)
      if (s0 + lane < s1) n_tab += (unsigned)((s1 - s0 - lane + 31) >> 5);
GPV_PRAGMA(unroll GPV_UNROLL)  // (2: two candidates in flight per lane; 1 measures the same, 3 slower)
      for (unsigned s = (unsigned)s0 + lane; s < (unsigned)s1; s += 32) {  // (suffix indices fit 32 bits)
        const int4 A = __ldg(tb.sf_hot + s);  // fs, nz4 | k << 8 | 8*b1 << 16, rb0..3, nzs0..3
        const int fk = (int)__byte_perm((unsigned)A.y, 0u, 0x4441);
        const int S = kp + fk;
        const int extra = Lx - (fp + A.x);
        bool slow = (unsigned)extra >= (unsigned)S;  // (always under defer_all: Lx < 0)
        int a = 0, b = 0, dP = 0, dS = 0;
        if (!slow) {
          if (R > 1) {  // branch-free: unused stage slots read the sentinel count
            // b = #{j < fk : cntb[rb_j] + j < extra}, the four tests as one byte-wise
            // subtraction: byte j of (extra + 128) - (cntb[rb_j] + j + 1) keeps bit 7 iff the
            // test holds (both sides < 128, so no borrow crosses a byte)
            // (bytes 1, 2 zero-extended by PRMT with a zero operand: one instruction each)
            const unsigned c0 = cntb[A.z & 0xff], c1 = cntb[__byte_perm((unsigned)A.z, 0u, 0x4441)];
            const unsigned c2 = cntb[__byte_perm((unsigned)A.z, 0u, 0x4442)], c3 = cntb[(unsigned)A.z >> 24];
            const unsigned w = __byte_perm(__byte_perm(c0, c1, 0x0040), __byte_perm(c2, c3, 0x0040), 0x5410) +
                               0x04030201u;  // bytes (c0, c1, c2, c3), each < 128
            const unsigned ge = ((unsigned)extra * 0x01010101u + 0x80808080u) - w;
            b = __popc(ge & 0x80808080u);  // (slots j >= fk read the sentinel count)
          } else {
            b = extra;
          }
          a = extra - b;
          // (no stage can exceed L layers here: every floor is <= L - extra, so the tables'
          // over-L bits are never set for a candidate's own promotion counts)
          GP_CHECK(!((pbad >> a) & 1));
          // byte b of the 40-bit zero-count word {A.y:A.w} (b <= 4): one PRMT
#ifdef GP_DEBUG_CHECKS
          GP_CHECK(b >= 0 && b <= 4 && b <= fk);
          if (!slow) GP_CHECK(a >= F.a_lo && a <= F.a_hi);  // the candidate's promotion count was tabulated
#endif
          const int nz = F.nzp[a] + (int)(__byte_perm((unsigned)A.w, (unsigned)A.y, (unsigned)b) & 0xff);
          if (nz > kDonations) slow = true;
          // zero-layer fix-up: each donation comes from the side holding the first maximum
          // (the prefix on ties: its stages come first); a donor must keep >= 1 layer
#if GPV_MERGE
          // the donors are the nz largest of the merge of the two non-increasing donor
          // sequences (prefix first on ties): common cases "all from one side" first
          if (nz > 0 && !slow) {
            const signed char* __restrict__ msr = tb.sf_ms + s * kMsStride + b * (kDonations + 1);
            const short* mpr = F.mp[a];
            const int mpl = mpr[nz - 1], ms0 = __ldg(msr);
            int last;
            if (mpl >= ms0) {
              dP = nz;
              last = mpl;
            } else {
              const int msl = __ldg(msr + nz - 1), mp0 = mpr[0];
              if (msl > mp0) {
                dS = nz;
                last = msl;
              } else {
#pragma unroll
                for (int i = 1; i <= kDonations; ++i)
                  if (i <= nz) dP += mpr[i - 1] >= __ldg(msr + nz - i) ? 1 : 0;
                dS = nz - dP;
                const int lp = dP > 0 ? mpr[dP - 1] : 127, ls = dS > 0 ? __ldg(msr + dS - 1) : 127;
                last = lp < ls ? lp : ls;
              }
            }
            if (last < 2) slow = true;
          }
#else
          for (int i = 0; i < nz && !slow; ++i) {
            const int mpv = F.mp[a][dP], msv = tb.sf_ms[s * kMsStride + b * (kDonations + 1) + dS];
            if ((mpv > msv ? mpv : msv) < 2) slow = true;
            if (mpv >= msv) ++dP;
            else ++dS;
          }
#endif
        }
        if (slow) {
          const long long key = pbase + s;
          const unsigned long long at = atomicAdd(slow_q, 1ULL);
          if (at < (unsigned long long)kSlowQueue) slow_q[1 + at] = (unsigned long long)key;
          --n_tab;
        } else {  // (no early exits: a flat if/else keeps the loop's reconvergence cheap)
#ifdef GP_DEBUG_CHECKS
          GP_CHECK(dP >= 0 && dP <= F.dm[a] && dS >= 0 && dS <= kDonations && S <= GP_MAX_STAGES);
#endif
          const double2 pa = F.pt[a][dP];
          const double2 sb = tb.sf_st[(b * (kDonations + 1) + dS) * nsuf32 + s];
          double mt = pa.x, mc = pa.y;
          if (sb.x > mt) mt = sb.x;
          if (sb.y > mc) mc = sb.y;
          if (mt < __longlong_as_double(0x7ff0000000000000LL)) {  // else memory-infeasible
            double tr = dtr;
            GP_CHECK(((unsigned)A.y >> 16) < 8 * kMaxJunction);
            if (R > 1) tr += *reinterpret_cast<const double*>(reinterpret_cast<const char*>(txs) + ((unsigned)A.y >> 16));
            // internal transfers of the suffix (t0, t1 | t2 planes, coalesced): absent terms are 0.0
            const double2 t01 = __ldg(reinterpret_cast<const double2*>(tb.sf_t) + s);
            tr += t01.x;
            tr += t01.y;
            tr += __ldg(tb.sf_t + (2u * (unsigned)nsuf32 + s));
            const double x = mt + fdk[fk] * mc + tr;  // fd[S], S = kp + fk
            if (DUMP && pbase + s >= rg.dump_lo && pbase + s < rg.dump_hi) rg.dump[pbase + s - rg.dump_lo] = x;
            ++feasible;
            if (x <= xthr) {  // within two ulps of the smallest so far (the key is formed only here)
              const long long d = __double_as_longlong(x) - b0;
              const long long key = pbase + s;
              if (d < 0) {
                k2 = d == -1 ? k1 : d == -2 ? k0 : LLONG_MAX;
                k1 = d == -1 ? k0 : LLONG_MAX;
                k0 = key;
                b0 += d;
                xthr = __longlong_as_double(b0 + 2);
              } else if (d == 1) {
                k1 = min(k1, key);
              } else if (d == 2) {
                k2 = min(k2, key);
              }
            }
          } else if (DUMP && pbase + s >= rg.dump_lo && pbase + s < rg.dump_hi) {
            rg.dump[pbase + s - rg.dump_lo] = mt;
          }
        }
      }
      __syncwarp();
      if (lane == 0 && p + 1 < p_end) prefix_advance_fast<R>(sp, P, kp);
    }
#if GPV_DYN
    unsigned long long nx = 0;
    if (lane == 0) nx = (unsigned long long)n_warps + atomicAdd(rg.work, 1ULL);
    it = (long long)__shfl_sync(0xffffffffu, nx, 0);
#endif
  }
  cp_async_wait_all();  // (a last middle-row prefetch may still be in flight)
  n_tab = __reduce_add_sync(0xffffffffu, n_tab);
  if (lane == 0) atomicAdd(&g_k1_fast_cnt[0], (unsigned long long)n_tab);
  NearMin nm{b0, {k0, k1, k2}, feasible};
  nm = nm_block_reduce<kK1Threads / 32>(nm);
  if (threadIdx.x == 0) partial[blockIdx.x] = nm;
}

// The candidates K1-fast deferred, scored by the generic eval_layout (rare; keys arrive
// in any order, so the summary merges them with nm_merge).
template <int R, bool DUMP = false>
__global__ void __launch_bounds__(kK1Threads) k1_deferred(TrainSpace sp, TrainTables tb,
                                                         const double2* __restrict__ blkf, int L,
                                                         const unsigned long long* __restrict__ slow_q,
                                                         NearMin* __restrict__ partial, ScanRange rg) {
  const unsigned long long cnt = slow_q[0];
  const long long n = (long long)min(cnt, (unsigned long long)kSlowQueue);
  NearMin m;
  nm_init(m);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long key = (long long)slow_q[1 + i];  // a rank
    Prefix<R> P;
    long long s;
    rank_decode<R>(sp, key, P, s);
    PrefixData<R> D;
    prefix_data<R>(sp, tb, blkf, P, D);
    double x;
    const bool ok = eval_layout<R, false>(sp, tb, blkf, L, D, tb.suf[s], x, nullptr, nullptr);
    if (DUMP && key >= rg.dump_lo && key < rg.dump_hi)
      rg.dump[key - rg.dump_lo] = ok ? x : __longlong_as_double(0x7ff0000000000000LL);
    if (ok) {
      NearMin o;
      o.b0 = __double_as_longlong(x);
      o.key[0] = key;
      o.key[1] = o.key[2] = LLONG_MAX;
      o.feasible = 1;
      nm_merge(m, o);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_k1_fast_cnt[1], (unsigned long long)n);
  m = nm_block_reduce(m);
  if (threadIdx.x == 0) partial[blockIdx.x] = m;
}

// Merge CTA summaries, pick the window's winner (keys are ranks) and decode its plan.
template <int R>
__device__ __forceinline__ void k1_finalize_body(const TrainSpace& sp, const TrainTables& tb,
                                                 const double2* __restrict__ blkf,
                                                 const BlockRec* __restrict__ blk, int L, int window,
                                                 const NearMin* __restrict__ partial, int n_partial,
                                                 TrainOut* __restrict__ out,
                                                 const unsigned long long* __restrict__ slow_q, const Scalars& sc,
                                                 const double* __restrict__ ceff, int mode) {
  NearMin m;
  nm_init(m);
  for (int i = threadIdx.x; i < n_partial; i += blockDim.x) nm_merge(m, partial[i]);
  m = nm_block_reduce(m);
  if (threadIdx.x != 0) return;
  double cost;
  const long long key = nm_winner(m, window, cost);
  out->best = Best{cost, key, m.feasible};
  out->overflow = slow_q && slow_q[0] > (unsigned long long)kSlowQueue;  // -> generic rescan
  out->nm_b0 = m.b0;
  for (int i = 0; i < 3; ++i) out->nm_rank[i] = m.key[i];
  out->n_stages = 0;
  if (key == LLONG_MAX) return;
  Prefix<R> P;
  long long s;
  rank_decode<R>(sp, key, P, s);
  PrefixData<R> D;
  prefix_data<R>(sp, tb, blkf, P, D);
  constexpr int NS = R * kMaxPerRun;
  int lay[NS], bis[NS];
  double x;
  eval_layout<R, true>(sp, tb, blkf, L, D, tb.suf[s], x, lay, bis);
  // mode 1 (product space): the first option combination in odometer order reaching the
  // layout's minimum — per stage the lowest tp whose total does not exceed M* = max over the
  // stages of their minimal totals (any such stage choice keeps the maximum at M*)
  double mstar = 0;
  for (int q = 0; q < NS; ++q)
    if (bis[q] >= 0) {
      const double v = tb.stage[(size_t)bis[q] * L + (lay[q] - 1)].x;
      if (v > mstar) mstar = v;
    }
  int n = 0;
  for (int q = 0; q < NS; ++q) {
    if (bis[q] < 0) continue;
    const BlockRec& br = blk[bis[q]];
    int o = tb.opt[(size_t)bis[q] * L + (lay[q] - 1)];
    if (mode == 1) {
      for (int oo = 0; oo < 4; ++oo) {
        double cmp, tpc, dpc;
        if (stage_option(br, lay[q], oo, sc, ceff[br.type], cmp, tpc, dpc) && cmp + tpc + dpc <= mstar) {
          o = oo;
          break;
        }
      }
    }
    const int tp = 1 << o;
    out->first[n] = br.start;
    out->count[n] = br.n;
    out->tp[n] = tp;
    out->dp[n] = br.n / tp;
    out->layers[n] = lay[q];
    ++n;
  }
  out->n_stages = n;
}

template <int R>
__global__ void __launch_bounds__(256) k1_finalize(TrainSpace sp, TrainTables tb,
                                                   const double2* __restrict__ blkf,
                                                   const BlockRec* __restrict__ blk, int L,
                                                   int window, const NearMin* __restrict__ partial,
                                                   int n_partial, TrainOut* __restrict__ out,
                                                   const unsigned long long* __restrict__ slow_q,
                                                   Scalars sc, const double* __restrict__ ceff, int mode) {
  k1_finalize_body<R>(sp, tb, blkf, blk, L, window, partial, n_partial, out, slow_q, sc, ceff, mode);
}

// ------------------------------------------------------- fused small-set path
// A scheduler / exhaustive batch holds many train sets whose whole space is a few thousand
// layouts; per-set launches of K2a..K2d, K1 and finalize would dominate. One CTA runs the
// complete pipeline of one such set (the same bodies as the per-set kernels, phases
// separated by CTA barriers), one launch per batch and type-run count.
struct SmallSet {
  TrainSpace sp;
  TrainTables tb;
  ScanRange rg;
  const BlockMeta* meta;
  const int* run_start;
  const int4* items;
  const int4* choices;
  BlockRec* blk;
  double2* blkf;
  double2* stage;
  int8_t* opt;
  double* tin;
  double* tx;
  double* fd;
  SufEnt* suf;
  NearMin* partial;
  TrainOut* out;
  int nblk, n_items, n_choices, mode;
};
constexpr long long kSmallLayouts = 1 << 12;  // spaces up to this size take the fused path

template <int R>
__global__ void __launch_bounds__(kK1Threads) k_train_small(const SmallSet* __restrict__ sets, Scalars sc,
                                                            const int* __restrict__ dtype,
                                                            const int* __restrict__ dmachine,
                                                            const double* __restrict__ dflops,
                                                            const double* __restrict__ dcap,
                                                            const double* __restrict__ links, int N,
                                                            const double* __restrict__ ceff, double numer,
                                                            int window) {
  const SmallSet& S = sets[blockIdx.x];
  const int L = sc.L;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int b = 0; b < S.nblk; ++b)  // K2a (CTA per block, sequentially)
    k2a_body(b, S.tb.ordered, S.meta, S.tb.pos, S.tb, S.blk, dtype, dmachine, dflops, dcap, links, N, L, sc.mb,
             S.fd, S.blkf);
  for (int it = wid; it < S.n_items; it += nw)  // K2b (warp per item)
    k2b_body(it, lane, S.tb.ordered, S.items, S.tb.pos, S.tb, S.sp, S.run_start, links, N, numer, S.tin, S.tx);
  __syncthreads();
  for (long long idx = threadIdx.x; idx < (long long)S.nblk * L; idx += blockDim.x)  // K2c
    k2c_body(idx, S.blk, sc, ceff, S.mode, S.stage, S.opt);
  for (int i = threadIdx.x; i < S.n_choices; i += blockDim.x)  // K2d
    k2d_body(i, S.choices, S.sp, S.tin, S.suf, S.sp.R - 1);
  __syncthreads();
  __shared__ Prefix<R> sP[kK1Threads / 32];
  __shared__ PrefixData<R> sD[kK1Threads / 32];
  NearMin nm = k1_scan_warps<R>(S.sp, S.tb, S.blkf, L, S.rg, wid, nw, sP[wid], sD[wid]);
  nm = nm_block_reduce(nm);
  if (threadIdx.x == 0) S.partial[0] = nm;
  __syncthreads();
  k1_finalize_body<R>(S.sp, S.tb, S.blkf, S.blk, L, window, S.partial, 1, S.out, nullptr, sc, ceff, S.mode);
}

// ===================================================================== host

namespace {

struct HostSpace {
  TrainSpace sp{};
  std::vector<int> ordered;
  std::vector<int> run_start;  // global offset of each run
  std::vector<int> pos;        // concatenated positions
  std::vector<int> pos_off;
  std::vector<BlockMeta> meta;
  std::vector<int4> items;
  std::vector<int4> choices;   // last-run choices (k, b1, b2, b3)
  int nblk = 0, tin_size = 0, tx_size = 0;
  long long total = 0;
  long long n_prefix = 0;
  std::vector<int> mgrp, gstart, gmach;  // machine groups of the canonical order
  bool exact_total = false;  // every partial FLOPS sum exact: K1-fast applies
  double flops_total = 0;    // allocate_layers' total (the same for every layout when exact)
  std::vector<int4> choices_m;  // choices of the middle run R - 2 (K1-fast's MidRow tables)
};

// choices (k, cut positions) of run r in run_compositions order (k ascending, cuts lexicographic)
static void run_choices(const TrainSpace& sp, int r, std::vector<int4>& out) {
  out.clear();
  const int nc = sp.nc[r];
  for (int k = 1; k <= sp.kmax[r]; ++k) {
    const int m = k - 1;
    if (nc < m) break;
    int c[3] = {0, 1, 2};
    while (true) {
      int4 ch = make_int4(k, 0, 0, 0);
      if (m > 0) ch.y = c[0] + 1;
      if (m > 1) ch.z = c[1] + 1;
      if (m > 2) ch.w = c[2] + 1;
      out.push_back(ch);
      int j = m - 1;
      while (j >= 0 && c[j] == nc - m + j) --j;
      if (j < 0) break;
      ++c[j];
      for (int t = j + 1; t < m; ++t) c[t] = c[t - 1] + 1;
    }
  }
}

// completion counts cnt / cntP of a TrainSpace whose per-run fields are set
static void space_counts(TrainSpace& sp) {
  std::memset(sp.cnt, 0, sizeof sp.cnt);
  std::memset(sp.cntP, 0, sizeof sp.cntP);
  for (int u = 0; u <= sp.max_stages; ++u) {
    sp.cnt[sp.R][u] = 1;
    sp.cntP[sp.R - 1][u] = 1;
  }
  for (int r = sp.R - 1; r >= 0; --r) {
    const int rem = sp.R - 1 - r;
    for (int u = 0; u <= sp.max_stages; ++u) {
      long long acc = 0, accP = 0;
      for (int k = 1; k <= sp.kmax[r]; ++k) {
        if (u + k + rem > sp.max_stages) break;
        acc += binom_small(sp.nc[r], k - 1) * sp.cnt[r + 1][u + k];
        if (r + 1 < sp.R) accP += binom_small(sp.nc[r], k - 1) * sp.cntP[r + 1][u + k];
      }
      sp.cnt[r][u] = acc;
      if (r + 1 < sp.R) sp.cntP[r][u] = accP;
    }
  }
}

// True when every partial sum of these devices' FLOPS is exactly representable: all are
// integer multiples of 2^e (e = the smallest trailing exponent) and sum / 2^e < 2^53.
static bool exact_flops_total(const gp_ctx* ctx, const std::vector<int>& ids, double* total) {
  int e_min = INT_MAX;
  for (int id : ids) {
    const double f = ctx->h_flops[id];
    if (!(f >= 0) || !std::isfinite(f)) return false;
    if (f == 0) continue;
    int ex;
    const double m = std::frexp(f, &ex);  // f = m * 2^ex, m in [0.5, 1)
    const unsigned long long mi = (unsigned long long)std::ldexp(m, 53);
    e_min = std::min(e_min, ex - 53 + __builtin_ctzll(mi));
  }
  double t = 0;
  if (e_min != INT_MAX) {
    unsigned long long units = 0;
    for (int id : ids) {
      const double q = std::ldexp(ctx->h_flops[id], -e_min);  // exact integer
      if (q >= 9007199254740992.0) return false;
      units += (unsigned long long)q;
      if (units >= (1ULL << 53)) return false;
    }
  }
  for (int id : ids) t += ctx->h_flops[id];
  *total = t;
  return true;
}

int build_space(gp_ctx* ctx, const int32_t* ids, int n, const gp_train_opts* o, HostSpace& h) {
  if (n <= 0) return set_error(GP_INVALID, "constrained_search requires a non-empty train set");
  if (o->max_stages_per_type < 1 || o->max_stages_per_type > kMaxPerRun)
    return set_error(GP_INVALID, "max_stages_per_type must lie in [1, 4] for the sm_100a kernel");
  h.ordered.assign(ids, ids + n);
  for (int id : h.ordered)
    if (id < 0 || id >= ctx->N) return set_error(GP_INVALID, "unknown device id " + std::to_string(id));
  // canonical_order (src/train_search.cpp:13-22)
  std::sort(h.ordered.begin(), h.ordered.end(), [&](int a, int b) {
    if (ctx->h_type[a] != ctx->h_type[b]) return ctx->h_type[a] < ctx->h_type[b];
    if (ctx->h_machine[a] != ctx->h_machine[b]) return ctx->h_machine[a] < ctx->h_machine[b];
    return a < b;
  });
  for (int i = 1; i < n; ++i)
    if (h.ordered[i] == h.ordered[i - 1])
      return set_error(GP_INVALID, "duplicate device id " + std::to_string(h.ordered[i]));
  // build_runs (src/train_search.cpp:30-50)
  const bool dev_gran = n <= o->device_granularity_limit;
  TrainSpace& sp = h.sp;
  sp.R = 0;
  for (int i = 0; i < n; ++i) {
    if (i == 0 || ctx->h_type[h.ordered[i]] != ctx->h_type[h.ordered[i - 1]]) {
      if (sp.R == GP_MAX_TYPES) return set_error(GP_INVALID, "too many gpu types");
      h.run_start.push_back(i);
      sp.R++;
    }
  }
  h.run_start.push_back(n);
  sp.n = n;
  sp.max_per_run = o->max_stages_per_type;
  sp.max_stages = std::min(ctx->sc.L, sp.R * o->max_stages_per_type);
  if (sp.max_stages > GP_MAX_STAGES) return set_error(GP_INVALID, "max_stages exceeds GP_MAX_STAGES");
  for (int r = 0; r < sp.R; ++r) {
    const int s0 = h.run_start[r], len = h.run_start[r + 1] - s0;
    sp.len[r] = len;
    h.pos_off.push_back((int)h.pos.size());
    h.pos.push_back(0);
    for (int i = 1; i < len; ++i) {
      const bool edge = ctx->h_machine[h.ordered[s0 + i]] != ctx->h_machine[h.ordered[s0 + i - 1]];
      if (dev_gran || edge) h.pos.push_back(i);
    }
    h.pos.push_back(len);
    sp.nc[r] = (int)(h.pos.size() - h.pos_off[r]) - 2;
    sp.kmax[r] = std::min(sp.max_per_run, len);
  }
  // completion counts: cnt over all runs, cntP over the prefix runs
  space_counts(sp);
  h.exact_total = exact_flops_total(ctx, h.ordered, &h.flops_total);
  h.mgrp.resize(n);
  for (int i = 0; i < n; ++i) {
    if (i == 0 || ctx->h_machine[h.ordered[i]] != ctx->h_machine[h.ordered[i - 1]]) {
      h.gstart.push_back(i);
      h.gmach.push_back(ctx->h_machine[h.ordered[i]]);
    }
    h.mgrp[i] = (int)h.gstart.size() - 1;
  }
  h.gstart.push_back(n);
  const bool any = sp.max_stages >= sp.R;
  h.total = any ? sp.cnt[0][0] : 0;
  h.n_prefix = any ? sp.cntP[0][0] : 0;
  // blocks, transfer items
  h.nblk = 0;
  h.tin_size = 0;
  h.tx_size = 0;
  for (int r = 0; r < sp.R; ++r) {
    const int nc = sp.nc[r], e = nc + 2;
    sp.blk_off[r] = h.nblk;
    for (int a = 0; a <= nc; ++a)
      for (int b = a + 1; b <= nc + 1; ++b) h.meta.push_back(BlockMeta{r, a, b, h.run_start[r]});
    h.nblk += (nc + 2) * (nc + 1) / 2;
    sp.tin_off[r] = h.tin_size;
    h.tin_size += e * e * e;
    for (int a = 0; a <= nc - 1; ++a)
      for (int b = a + 1; b <= nc; ++b)
        for (int c = b + 1; c <= nc + 1; ++c) h.items.push_back(make_int4(r, a, b, c));
    sp.tx_off[r] = h.tx_size;
    if (r + 1 < sp.R) {
      const int e2 = sp.nc[r + 1] + 2;
      h.tx_size += e * e2;
      for (int a = 0; a <= nc; ++a)
        for (int c = 1; c <= sp.nc[r + 1] + 1; ++c) h.items.push_back(make_int4(r, a, 0, -c));
    }
  }
  // last-run choices in run_compositions order: k ascending, cut indices lexicographic
  run_choices(sp, sp.R - 1, h.choices);
  sp.n_suf = (int)h.choices.size();
  if (sp.R >= 2) run_choices(sp, sp.R - 2, h.choices_m);
  return GP_OK;
}
// Host twin of prefix_decode's base (rank of a prefix's first layout).
template <int R>
long long prefix_base_host(const TrainSpace& sp, long long p) {
  Prefix<R> P;
  return prefix_decode<R>(sp, p, P);
}

long long prefix_base(const TrainSpace& sp, long long p) {
  switch (sp.R) {
    case 1: return 0;
    case 2: return prefix_base_host<2>(sp, p);
    case 3: return prefix_base_host<3>(sp, p);
    case 4: return prefix_base_host<4>(sp, p);
    default: return prefix_base_host<8>(sp, p);
  }
}

// rank (of sp's enumeration order) -> (prefix, suffix): the last prefix whose base <= rank.
void rank_split(const TrainSpace& sp, long long rank, long long& p, long long& s) {
  const bool any = sp.max_stages >= sp.R;
  const long long total = any ? sp.cnt[0][0] : 0, n_prefix = any ? sp.cntP[0][0] : 0;
  if (rank >= total) {
    p = n_prefix;
    s = 0;
    return;
  }
  long long lo = 0, hi = n_prefix - 1;
  while (lo < hi) {
    const long long mid = lo + (hi - lo + 1) / 2;
    if (prefix_base(sp, mid) <= rank) lo = mid;
    else hi = mid - 1;
  }
  p = lo;
  s = rank - prefix_base(sp, lo);
}
void rank_split(const HostSpace& h, long long rank, long long& p, long long& s) { rank_split(h.sp, rank, p, s); }

template <typename T>
T* carve(char*& p, size_t count) {
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
  T* r = reinterpret_cast<T*>(p);
  p += sizeof(T) * count;
  return r;
}

// What one K1 launch scans: ranks [lo, hi) of the reference order, with K1-fast or the
// generic K1. dump (test hook): per_step of the ranks [dump_lo, dump_hi).
struct ScanSpec {
  long long lo = 0, hi = 0;
  bool fast = false;
  double* dump = nullptr;
  long long dump_lo = 0, dump_hi = 0;
  bool defer_all = false;
};

template <int R>
int launch_scan(gp_ctx* ctx, const HostSpace& h, const TrainTables& tb, const double2* blkf,
                const BlockRec* blk, int window, const ScanSpec& sc, NearMin* partial,
                int max_blocks, TrainOut* d_out, cudaStream_t stream, int mode,
                unsigned long long* slow_q) {
  const bool fast = sc.fast;
  const TrainSpace& sp = h.sp;
  ScanRange rg{};
  rg.dump = sc.dump;
  rg.dump_lo = sc.dump_lo;
  rg.dump_hi = sc.dump_hi;
  rank_split(sp, sc.lo, rg.p_lo, rg.s_lo);
  rank_split(sp, sc.hi, rg.p_hi, rg.s_hi);
  const char* defer_env = std::getenv("GPLAN_K1_DEFER_ALL");
  rg.defer_all = sc.defer_all || (defer_env && defer_env[0] == '1');
  rg.n_pref = rg.p_hi - rg.p_lo + (rg.s_hi > 0 ? 1 : 0);
  const int threads = kK1Threads;
  static std::once_flag occ_once;  // occupancy of the two scan kernels (shared by all contexts)
  static int occ_tab[2][5];
  std::call_once(occ_once, [] {
    const void* fk[5] = {nullptr, (const void*)k1_layout_scan_fast<1>, (const void*)k1_layout_scan_fast<2>,
                         (const void*)k1_layout_scan_fast<3>, (const void*)k1_layout_scan_fast<4>};
    const void* gk[5] = {nullptr, (const void*)k1_layout_scan<1>, (const void*)k1_layout_scan<2>,
                         (const void*)k1_layout_scan<3>, (const void*)k1_layout_scan<4>};
    for (int r = 1; r <= 4; ++r) {
      int o = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fk[r], kK1Threads, 0);
      occ_tab[1][r] = std::max(1, o);
      o = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, gk[r], kK1Threads, 0);
      occ_tab[0][r] = std::max(1, o);
    }
  });
  const int occ = occ_tab[fast ? 1 : 0][R];
  const long long warps_total = (long long)ctx->num_sms * occ * (threads / 32);
  rg.chunk = std::max(1LL, rg.n_pref / (warps_total * (fast && GPV_DYN ? GPV_ITEMS : 6)));
  // K1-fast: a work item starts with a prefix decode and, when its front differs from the
  // warp's last one, a front-table rebuild; keep items long enough to amortise both
  if (fast) rg.chunk = std::max<long long>(rg.chunk, GPV_MINCHUNK);
  // generic scan of a space with fewer than 32 suffixes per prefix on average: one prefix per
  // lane (gs = 1) — the serial prefix decode and tabulation then run on all 32 lanes at once,
  // and a handful of suffixes per lane follows (gs = 32: one prefix per warp, lanes over its
  // suffixes). GPLAN_K1_UNGROUPED=1 / GPLAN_K1_GROUP=4: the other layouts (tests, A/B).
  int gs = 32;
  if (!fast && R > 1 && !std::getenv("GPLAN_K1_UNGROUPED") && h.total < 32 * std::max(1LL, h.n_prefix)) {
    const char* ge = std::getenv("GPLAN_K1_GROUP");
    gs = ge && std::atoi(ge) == 4 ? 4 : 1;
    const long long G = 32 / gs;
    rg.chunk = (rg.chunk + G - 1) / G * G;
  }
  rg.work = slow_q ? slow_q + 1 + kSlowQueue : nullptr;
  const long long n_items = (rg.n_pref + rg.chunk - 1) / rg.chunk;
  long long blocks = (n_items + (threads / 32) - 1) / (threads / 32);
  blocks = std::max(1LL, std::min(blocks, std::min((long long)max_blocks, (long long)ctx->num_sms * occ)));
  int n_partial = (int)blocks;
  const int L = ctx->sc.L;
  if (sc.hi > sc.lo) {
    if (fast) {
      GP_CUDA(cudaMemsetAsync(slow_q, 0, sizeof(unsigned long long), stream));
      GP_CUDA(cudaMemsetAsync(slow_q + 1 + kSlowQueue, 0, sizeof(unsigned long long), stream));
      if (sc.dump) {
        k1_layout_scan_fast<R, true><<<(int)blocks, threads, 0, stream>>>(h.sp, tb, blkf, L, rg, partial, slow_q);
        k1_deferred<R, true><<<kDeferBlocks, threads, 0, stream>>>(h.sp, tb, blkf, L, slow_q, partial + blocks, rg);
      } else {
        k1_layout_scan_fast<R><<<(int)blocks, threads, 0, stream>>>(h.sp, tb, blkf, L, rg, partial, slow_q);
        k1_deferred<R><<<kDeferBlocks, threads, 0, stream>>>(h.sp, tb, blkf, L, slow_q, partial + blocks, rg);
      }
      n_partial += kDeferBlocks;
      ctx->launches += 2;
    } else if (gs < 32) {  // few suffixes per prefix: groups of gs lanes, G prefixes in lockstep
      auto go = [&](auto kern) { kern<<<(int)blocks, threads, 0, stream>>>(h.sp, tb, blkf, L, rg, partial); };
      if (gs == 1) sc.dump ? go(k1_layout_scan_grouped<R, 1, true>) : go(k1_layout_scan_grouped<R, 1>);
      else sc.dump ? go(k1_layout_scan_grouped<R, 4, true>) : go(k1_layout_scan_grouped<R, 4>);
      ctx->launches++;
    } else {
      if (sc.dump) k1_layout_scan<R, true><<<(int)blocks, threads, 0, stream>>>(h.sp, tb, blkf, L, rg, partial);
      else k1_layout_scan<R><<<(int)blocks, threads, 0, stream>>>(h.sp, tb, blkf, L, rg, partial);
      ctx->launches++;
    }
  } else {
    n_partial = 0;
  }
  k1_finalize<R><<<1, 256, 0, stream>>>(h.sp, tb, blkf, blk, L, window, partial, n_partial, d_out,
                                        fast && sc.hi > sc.lo ? slow_q : nullptr, ctx->sc, ctx->d_ceff, mode);
  ctx->launches++;
  GP_CUDA(cudaGetLastError());
  return GP_OK;
}

}  // namespace

// ---- product-space bookkeeping (enumerate_train_candidates, src/train_search.cpp:179-216):
// the number of candidates = sum over layouts of prod_s |tp_dp_options(block_s)|, and the
// candidate index of a (layout, option picks). Pure enumeration metadata (no cost model).
namespace {
struct CandMeta {
  const HostSpace* h;
  const gp_ctx* ctx;
  std::vector<std::vector<int>> wt;  // per run: options of block [a, b), (nc+2)^2 table
  std::vector<std::vector<int>> tps;  // per run: option tp values, 4 per block
  void init() {
    const TrainSpace& sp = h->sp;
    wt.assign(sp.R, {});
    tps.assign(sp.R, {});
    for (int r = 0; r < sp.R; ++r) {
      const int e = sp.nc[r] + 2;
      const int* P = h->pos.data() + h->pos_off[r];
      wt[r].assign(e * e, 0);
      tps[r].assign(e * e * 4, 0);
      for (int a = 0; a + 1 < e; ++a) {
        // per-machine run lengths of the blocks starting at a, extended one position at a time
        int per_machine = 0, run = 0;
        const int s0 = h->run_start[r] + P[a];
        int i = s0;
        for (int b = a + 1; b < e; ++b) {
          const int s1 = h->run_start[r] + P[b];
          for (; i < s1; ++i) {
            run = (i > s0 && ctx->h_machine[h->ordered[i]] == ctx->h_machine[h->ordered[i - 1]]) ? run + 1 : 1;
            per_machine = std::max(per_machine, run);
          }
          int n = 0;
          for (int tp = 1; tp <= 8; tp *= 2)
            if (tp <= per_machine && (s1 - s0) % tp == 0) tps[r][(a * e + b) * 4 + n++] = tp;
          wt[r][a * e + b] = n;
        }
      }
    }
  }
  // options of the block [a, b) (position indices) of run r
  int w(int r, int a, int b, int* tp_out = nullptr) const {
    const int e = h->sp.nc[r] + 2;
    const int n = wt[r][a * e + b];
    if (tp_out)
      for (int j = 0; j < n; ++j) tp_out[j] = tps[r][(a * e + b) * 4 + j];
    return n;
  }
  // sum over cut combinations of run r with k blocks of the product of block weights
  long long G(int r, int k) const {
    const int nc = h->sp.nc[r];
    std::vector<std::vector<long long>> F(k + 1, std::vector<long long>(nc + 2, 0));
    F[0][0] = 1;
    for (int j = 0; j < k; ++j)
      for (int i = 0; i <= nc + 1; ++i) {
        if (!F[j][i]) continue;
        for (int i2 = i + 1; i2 <= nc + 1; ++i2) {
          if (j + 1 < k && i2 == nc + 1) continue;  // only the last block ends at the run end
          if (j + 1 == k && i2 != nc + 1) continue;
          F[j + 1][i2] += F[j][i] * w(r, i, i2);
        }
      }
    return F[k][nc + 1];
  }
};
}  // namespace

int train_candidates_meta(gp_ctx* ctx, const int32_t* ids, int n, const gp_train_result* res,
                          const int32_t* stage_devices, long long* count, long long* index) {
  HostSpace h;
  gp_train_opts o{4, 16};
  int rc = build_space(ctx, ids, n, &o, h);
  if (rc) return rc;
  const TrainSpace& sp = h.sp;
  CandMeta cm{&h, ctx, {}, {}};
  cm.init();
  std::vector<std::vector<long long>> W(sp.R + 1, std::vector<long long>(sp.max_stages + 2, 0));
  std::vector<std::vector<long long>> Gk(sp.R, std::vector<long long>(kMaxPerRun + 1, 0));
  for (int r = 0; r < sp.R; ++r)
    for (int k = 1; k <= sp.kmax[r] && k - 1 <= sp.nc[r]; ++k) Gk[r][k] = cm.G(r, k);
  for (int u = 0; u <= sp.max_stages; ++u) W[sp.R][u] = 1;
  for (int r = sp.R - 1; r >= 0; --r)
    for (int u = 0; u <= sp.max_stages; ++u) {
      long long acc = 0;
      for (int k = 1; k <= sp.kmax[r]; ++k) {
        if (u + k + (sp.R - 1 - r) > sp.max_stages) break;
        acc += Gk[r][k] * W[r + 1][u + k];
      }
      W[r][u] = acc;
    }
  *count = sp.max_stages >= sp.R ? W[0][0] : 0;
  *index = -1;
  if (!res || !res->found) return GP_OK;
  // the winner's blocks per run, as position indices
  long long before = 0, pick_index = 0, radix = 1, pw = 1;  // pw: weight of the chosen earlier runs
  int u = 0, st = 0;
  for (int r = 0; r < sp.R; ++r) {
    const int* P = h.pos.data() + h.pos_off[r];
    const int nc = sp.nc[r], base = h.run_start[r];
    std::vector<int> idx{0};
    while (st < res->n_stages && res->stage[st].first < h.run_start[r + 1]) {
      const int end = res->stage[st].first + res->stage[st].count - base;
      int pi = 0;
      while (pi <= nc + 1 && P[pi] != end) ++pi;
      idx.push_back(pi);
      int tps[4];
      const int nw = cm.w(r, idx[idx.size() - 2], pi, tps);
      int pk = 0;
      while (pk < nw && tps[pk] != res->stage[st].tp) ++pk;
      pick_index += pk * radix;
      radix *= nw;
      ++st;
    }
    const int k = (int)idx.size() - 1;
    for (int k2 = 1; k2 < k; ++k2) before += pw * Gk[r][k2] * W[r + 1][u + k2];
    // combinations of k-1 cut indices before the winner's, lexicographically
    std::vector<int> c(k + 1);
    c[0] = 0;
    c[k] = nc + 1;
    for (int j = 1; j < k; ++j) c[j] = j;
    while (true) {
      bool same = true;
      for (int j = 1; j < k; ++j) same &= c[j] == idx[j];
      if (same) break;
      long long wt = 1;
      for (int j = 0; j < k; ++j) wt *= cm.w(r, c[j], c[j + 1]);
      before += pw * wt * W[r + 1][u + k];
      int j = k - 1;  // next combination (lexicographic over c[1..k-1] in [1, nc])
      while (j >= 1 && c[j] == nc - (k - 1 - j)) --j;
      if (j < 1) break;
      ++c[j];
      for (int j2 = j + 1; j2 < k; ++j2) c[j2] = c[j2 - 1] + 1;
    }
    for (int j = 0; j < k; ++j) pw *= cm.w(r, idx[j], idx[j + 1]);
    u += k;
  }
  (void)stage_devices;
  *index = before + pick_index;
  return GP_OK;
}

int train_space(gp_ctx* ctx, const int32_t* ids, int n, const gp_train_opts* o, int64_t* layouts) {
  HostSpace h;
  int rc = build_space(ctx, ids, n, o, h);
  if (rc) return rc;
  *layouts = h.total;
  return GP_OK;
}


// A train set whose enumeration metadata is resident on the device
// (gp_train_prepare); gp_train_launch builds the K2 tables and scans a range.
struct PreparedTrain {
  HostSpace h;
  int* d_ordered = nullptr;
  int* d_pos = nullptr;
  int* d_run_start = nullptr;
  BlockMeta* d_meta = nullptr;
  int4* d_items = nullptr;
  int4* d_choices = nullptr;
  int4* d_choices_m = nullptr;  // middle-run choices (K1-fast)
  SufEnt* d_sufm = nullptr;     // middle-run choice table
  MidRow* d_mid = nullptr;
  unsigned long long* d_cntb_mid = nullptr;
  int* d_mgrp = nullptr;
  int* d_gstart = nullptr;
  int* d_gmach = nullptr;
  BlockRec* d_blk = nullptr;
  double2* d_blkf = nullptr;
  double2* d_stage = nullptr;
  int8_t* d_opt = nullptr;
  double* d_tin = nullptr;
  double* d_tx = nullptr;
  double* d_fd = nullptr;
  SufEnt* d_suf = nullptr;
  double2* d_blk_sh = nullptr;
  int4* d_sf_hot = nullptr;
  double* d_sf_t = nullptr;
  signed char* d_sf_ms = nullptr;
  double2* d_sf_st = nullptr;
  int* d_nzs_max = nullptr;
  NearMin* d_partial = nullptr;
  TrainOut* d_out = nullptr;
  int max_blocks = 0;
  int L = 0;
  long long lo = 0, hi = 0;
  int window = 0;
  int mode = 0;  // 0: constrained_search; 1: product space (enumerate_train_candidates)
  bool launched = false;
  long long nm[4] = {kInfBits, LLONG_MAX, LLONG_MAX, LLONG_MAX};  // NearMin of the last collect (ranks)
};

// GPLAN_PROFILE=1: memo hits / scanned sets / scanned layouts (stderr at exit)
struct MemoStats {  // (updated from the per-device threads of train_batch: atomics)
  std::atomic<long long> hits{0}, scans{0}, layouts{0};
  std::atomic<long long> size_sets[12] = {}, size_layouts[12] = {};  // scanned sets by log10(layouts)
  AtomicD ph[5];  // train_batch_run: build, carve+upload, launch, wait, fill
  std::atomic<unsigned long long> fast_cnt[2] = {{0}, {0}};
  void poll() {  // after a synchronisation
    if (!std::getenv("GPLAN_PROFILE")) return;
    unsigned long long c[2] = {0, 0};
    cudaMemcpyFromSymbol(c, g_k1_fast_cnt, sizeof c);
    fast_cnt[0] = c[0];
    fast_cnt[1] = c[1];
  }
  ~MemoStats() {
    if (std::getenv("GPLAN_PROFILE"))
      std::fprintf(stderr, "k1 fast: %llu candidates from tables, %llu by the generic fallback\n",
                   fast_cnt[0].load(), fast_cnt[1].load());
    if (std::getenv("GPLAN_PROFILE"))
      std::fprintf(stderr, "train memo: %lld hits, %lld scanned sets, %lld scanned layouts; batch phases: "
                   "build %.3f s, carve+upload %.3f s, launch %.3f s, wait %.3f s, fill %.3f s\n", hits.load(),
                   scans.load(), layouts.load(), (double)ph[0], (double)ph[1], (double)ph[2], (double)ph[3],
                   (double)ph[4]);
    if (std::getenv("GPLAN_PROFILE"))
      for (int b = 0; b < 12; ++b)
        if (size_sets[b].load())
          std::fprintf(stderr, "train sets of 1e%d..1e%d layouts: %lld sets, %lld layouts\n", b, b + 1,
                       size_sets[b].load(), size_layouts[b].load());
  }
} g_memo_stats;

static PreparedTrain*& prepared(gp_ctx* ctx) {
  return reinterpret_cast<PreparedTrain*&>(ctx->train_state);
}

void train_state_free(gp_ctx* ctx) {
  delete prepared(ctx);
  prepared(ctx) = nullptr;
}

// words of one middle-run rank-count row: the last run's blocks, 8 per word
static int cntb_words(const HostSpace& h) {
  const int e = h.sp.nc[h.sp.R - 1] + 2;
  return (e * (e - 1) / 2 + 7) / 8;
}

// ---- layout of one prepared train set in a device arena: the inputs section
// (copied from host) first, then the tables the kernels build.
static size_t input_bytes(const HostSpace& h) {
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += ((b + 255) & ~size_t(255)) + 256; };
  add(sizeof(int) * h.sp.n);
  add(sizeof(int) * h.pos.size());
  add(sizeof(int) * h.run_start.size());
  add(sizeof(BlockMeta) * h.meta.size());
  add(sizeof(int4) * h.items.size());
  add(sizeof(int4) * h.choices.size());
  add(sizeof(int4) * h.choices_m.size());
  add(sizeof(int) * h.mgrp.size());
  add(sizeof(int) * h.gstart.size());
  add(sizeof(int) * h.gmach.size());
  return bytes;
}

static size_t table_bytes(const HostSpace& h, int L, int max_blocks) {
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += ((b + 255) & ~size_t(255)) + 256; };
  add(sizeof(BlockRec) * h.nblk);
  add(sizeof(double2) * h.nblk);
  add(sizeof(double2) * (size_t)h.nblk * L);
  add(sizeof(int8_t) * (size_t)h.nblk * L);
  add(sizeof(double) * (h.tin_size + 1));
  add(sizeof(double) * (h.tx_size + 1));
  add(sizeof(double) * (GP_MAX_STAGES + 1));
  add(sizeof(SufEnt) * (h.choices.size() + 1));
  add(sizeof(SufEnt) * (h.choices_m.size() + 1));
  add(sizeof(MidRow) * (h.choices_m.size() + 1));
  add(sizeof(unsigned long long) * (h.choices_m.size() + 1) * cntb_words(h));
  add(sizeof(double2) * h.nblk);
  const size_t nsf = h.choices.size() + 1;
  add(sizeof(int4) * nsf);
  add(sizeof(double) * 4 * nsf);
  add((size_t)kMsStride * nsf);
  add(sizeof(double2) * 5 * (kDonations + 1) * nsf);
  add(sizeof(int) * (3 + 5 * (L + 1)));
  add(sizeof(NearMin) * (max_blocks + kDeferBlocks));
  return bytes;
}

// Carves the inputs at *in (device) and stages them into *hst (pinned host) at the same
// offsets relative to `in_base`/`h_base`; then carves the tables at *tab.
static void carve_prepared(PreparedTrain& P, char*& in, char*& tab, char* in_base, char* h_base) {
  const HostSpace& h = P.h;
  auto stage = [&](const void* src, size_t sz, void* dptr) {
    if (sz) std::memcpy(h_base + ((char*)dptr - in_base), src, sz);
  };
  P.d_ordered = carve<int>(in, h.sp.n);
  stage(h.ordered.data(), sizeof(int) * h.sp.n, P.d_ordered);
  P.d_pos = carve<int>(in, h.pos.size());
  stage(h.pos.data(), sizeof(int) * h.pos.size(), P.d_pos);
  P.d_run_start = carve<int>(in, h.run_start.size());
  stage(h.run_start.data(), sizeof(int) * h.run_start.size(), P.d_run_start);
  P.d_meta = carve<BlockMeta>(in, h.meta.size());
  stage(h.meta.data(), sizeof(BlockMeta) * h.meta.size(), P.d_meta);
  P.d_items = carve<int4>(in, h.items.size());
  stage(h.items.data(), sizeof(int4) * h.items.size(), P.d_items);
  P.d_choices = carve<int4>(in, h.choices.size());
  stage(h.choices.data(), sizeof(int4) * h.choices.size(), P.d_choices);
  P.d_choices_m = carve<int4>(in, h.choices_m.size());
  stage(h.choices_m.data(), sizeof(int4) * h.choices_m.size(), P.d_choices_m);
  P.d_mgrp = carve<int>(in, h.mgrp.size());
  stage(h.mgrp.data(), sizeof(int) * h.mgrp.size(), P.d_mgrp);
  P.d_gstart = carve<int>(in, h.gstart.size());
  stage(h.gstart.data(), sizeof(int) * h.gstart.size(), P.d_gstart);
  P.d_gmach = carve<int>(in, h.gmach.size());
  stage(h.gmach.data(), sizeof(int) * h.gmach.size(), P.d_gmach);
  P.d_blk = carve<BlockRec>(tab, h.nblk);
  P.d_blkf = carve<double2>(tab, h.nblk);
  P.d_stage = carve<double2>(tab, (size_t)h.nblk * P.L);
  P.d_opt = carve<int8_t>(tab, (size_t)h.nblk * P.L);
  P.d_tin = carve<double>(tab, h.tin_size + 1);
  P.d_tx = carve<double>(tab, h.tx_size + 1);
  P.d_fd = carve<double>(tab, GP_MAX_STAGES + 1);
  P.d_suf = carve<SufEnt>(tab, h.choices.size() + 1);
  P.d_sufm = carve<SufEnt>(tab, h.choices_m.size() + 1);
  P.d_mid = carve<MidRow>(tab, h.choices_m.size() + 1);
  P.d_cntb_mid = carve<unsigned long long>(tab, (h.choices_m.size() + 1) * cntb_words(h));
  P.d_blk_sh = carve<double2>(tab, h.nblk);
  const size_t nsf = h.choices.size() + 1;
  P.d_sf_hot = carve<int4>(tab, nsf);
  P.d_sf_t = carve<double>(tab, 4 * nsf);
  P.d_sf_ms = carve<signed char>(tab, (size_t)kMsStride * nsf);
  P.d_sf_st = carve<double2>(tab, 5 * (kDonations + 1) * nsf);
  P.d_nzs_max = carve<int>(tab, 3 + 5 * (P.L + 1));
  P.d_partial = carve<NearMin>(tab, P.max_blocks + kDeferBlocks);
}

static double sum_stages(const HostSpace& h) {
  double tot[GP_MAX_TYPES + 1][GP_MAX_STAGES + 1] = {};
  const TrainSpace& sp = h.sp;
  for (int r = sp.R - 1; r >= 0; --r)
    for (int u = 0; u <= sp.max_stages; ++u) {
      double acc = 0;
      for (int k = 1; k <= sp.kmax[r]; ++k) {
        if (u + k + (sp.R - 1 - r) > sp.max_stages) break;
        const double c = (double)binom_small(sp.nc[r], k - 1);
        acc += c * ((double)k * (double)sp.cnt[r + 1][u + k] + tot[r + 1][u + k]);
      }
      tot[r][u] = acc;
    }
  return h.total ? tot[0][0] : 0;
}

// Device-side table view of a prepared train set.
static TrainTables prepared_tables(const gp_ctx* ctx, const PreparedTrain& P) {
  TrainTables tb{};
  tb.ordered = P.d_ordered;
  tb.mgrp = P.d_mgrp;
  tb.gstart = P.d_gstart;
  tb.gmach = P.d_gmach;
  tb.mlinks = ctx->d_mlinks;
  tb.M = ctx->M;
  tb.pos = P.d_pos;
  tb.blk = P.d_blk;
  tb.stage = P.d_stage;
  tb.opt = P.d_opt;
  tb.tin = P.d_tin;
  tb.tx = P.d_tx;
  tb.fd_coef = P.d_fd;
  tb.suf = P.d_suf;
  tb.blk_sh = P.d_blk_sh;
  tb.sf_hot = P.d_sf_hot;
  tb.sf_t = P.d_sf_t;
  tb.sf_ms = P.d_sf_ms;
  tb.sf_st = P.d_sf_st;
  tb.nzs_max = P.d_nzs_max;
  tb.mid = P.d_mid;
  tb.cntb_mid = P.d_cntb_mid;
  tb.cw = cntb_words(P.h);
  tb.n_mid = (int)P.h.choices_m.size();
  for (int r = 0; r < P.h.sp.R; ++r) tb.pos_off[r] = P.h.pos_off[r];
  return tb;
}

// Enqueues K2 + K1 + finalize for P over ranks [lo, hi) on `stream` (asynchronous).
// dump (test hook, gp_debug_layout_costs): per_step of ranks [dump_lo, dump_hi).
static int launch_prepared(gp_ctx* ctx, PreparedTrain& P, int window, long long lo, long long hi,
                           cudaStream_t stream, bool timing, bool force_generic = false, int lane = -1,
                           double* dump = nullptr, bool* used_fast = nullptr, bool defer_all = false,
                           long long dump_lo = 0, long long dump_hi = 0) {
  const HostSpace& h = P.h;
  if (lo < 0) lo = 0;
  if (hi < 0 || hi > h.total) hi = h.total;
  if (lo > hi) lo = hi;
  P.lo = lo;
  P.hi = hi;
  P.window = window;
  P.launched = true;
  if (h.total == 0 || lo == hi) return GP_OK;  // std::nullopt
  const int L = ctx->sc.L;
  TrainTables tb = prepared_tables(ctx, P);
  const char* generic_env = std::getenv("GPLAN_K1_GENERIC");
  const int R = h.sp.R;
  // (layer counts are tabulated as signed bytes: L <= 127; small spaces: the generic scan —
  // the fast path's extra table launches would dominate)
  // K1-fast puts the last run's choices on the lanes of a warp and pays a table merge per
  // prefix: with fewer than kFastMinSuffixes last-run choices per prefix on average (a last
  // type run of one or two machines) most lanes idle and the generic scan is faster
  const int nlast = (h.sp.nc[R - 1] + 2) * (h.sp.nc[R - 1] + 1) / 2;
  const bool fast = h.exact_total && h.total >= (1LL << 20) && L <= 127 && nlast <= kSentinelBlock &&
                    h.sp.nc[R - 1] + 2 <= kMaxJunction && h.total >= kFastMinSuffixes * h.n_prefix &&
                    !force_generic && !(generic_env && generic_env[0] == '1');
  if (used_fast) *used_fast = fast;
  unsigned long long*& slow_q = lane < 0 ? ctx->d_slow : ctx->d_slow_lane[lane];
  if (fast && !slow_q) GP_CUDA(cudaMalloc(&slow_q, sizeof(unsigned long long) * (2 + kSlowQueue)));
  if (timing) GP_CUDA(cudaEventRecord(ctx->ev[0], stream));
  // ---- K2: per-train-set tables
  k2a_block_stats<<<h.nblk, 256, 0, stream>>>(P.d_ordered, P.d_meta, P.d_pos, tb, P.d_blk, ctx->d_type,
                                              ctx->d_machine, ctx->d_flops, ctx->d_hbm_cap, ctx->d_links,
                                              ctx->N, L, ctx->sc.mb, P.d_fd, P.d_blkf);
  ctx->launches++;
  if (!h.items.empty()) {
    const int warps_per_block = 8;
    const int grid = (int)((h.items.size() + warps_per_block - 1) / warps_per_block);
    k2b_transfers<<<grid, 32 * warps_per_block, 0, stream>>>(
        P.d_ordered, P.d_items, (int)h.items.size(), P.d_pos, tb, h.sp, P.d_run_start, ctx->d_links, ctx->N,
        ctx->sc.tokens > 0 ? ctx->sc.act_tok_h2 : 0.0, P.d_tin, P.d_tx);
    ctx->launches++;
  }
  {
    const long long cnt = (long long)h.nblk * L;
    k2c_stage_table<<<(int)((cnt + 255) / 256), 256, 0, stream>>>(P.d_blk, h.nblk, ctx->sc, ctx->d_ceff,
                                                                 P.mode, P.d_stage, P.d_opt);
    const int ns = (int)h.choices.size();
    k2d_suffix_table<<<(ns + 255) / 256, 256, 0, stream>>>(P.d_choices, ns, h.sp, P.d_tin, P.d_suf, R - 1);
    ctx->launches += 2;
    if (fast) {
      k2e_block_shares<<<(h.nblk + 255) / 256, 256, 0, stream>>>(P.d_blkf, h.nblk, h.flops_total, P.d_blk_sh);
      GP_CUDA(cudaMemsetAsync(P.d_nzs_max, 0, (3 + 5 * (L + 1)) * sizeof(int), stream));
      k2f_suffix_fast<<<(ns + 127) / 128, 128, 0, stream>>>(P.d_suf, ns, P.d_blk_sh, P.d_stage, L,
                                                           h.sp.blk_off[R - 1], P.d_sf_hot,
                                                           P.d_sf_t, P.d_sf_ms, P.d_sf_st, P.d_nzs_max);
      if (R >= 2) {  // the middle run's rows (K2d on run R - 2, then K2m)
        const int nm = (int)h.choices_m.size();
        const int e_last = h.sp.nc[R - 1] + 2;
        k2d_suffix_table<<<(nm + 255) / 256, 256, 0, stream>>>(P.d_choices_m, nm, h.sp, P.d_tin, P.d_sufm, R - 2);
        k2m_middle_rows<<<(nm + 127) / 128, 128, 0, stream>>>(P.d_sufm, nm, P.d_blk_sh, P.d_stage, L,
                                                             h.sp.blk_off[R - 1], e_last * (e_last - 1) / 2,
                                                             cntb_words(h), P.d_mid, P.d_cntb_mid);
        ctx->launches += 2;
      }
      ctx->launches += 2;
    }
  }
  GP_CUDA(cudaGetLastError());
  if (timing) GP_CUDA(cudaEventRecord(ctx->ev[1], stream));
  // ---- K1: layout scan over [lo, hi)
  ScanSpec sc;
  sc.lo = lo;
  sc.hi = hi;
  sc.fast = fast;
  sc.dump = dump;
  sc.dump_lo = dump_lo;
  sc.dump_hi = dump_hi;
  sc.defer_all = defer_all;
  int rc;
  if (R == 1) rc = launch_scan<1>(ctx, h, tb, P.d_blkf, P.d_blk, window, sc, P.d_partial, P.max_blocks, P.d_out, stream, P.mode, slow_q);
  else if (R == 2) rc = launch_scan<2>(ctx, h, tb, P.d_blkf, P.d_blk, window, sc, P.d_partial, P.max_blocks, P.d_out, stream, P.mode, slow_q);
  else if (R == 3) rc = launch_scan<3>(ctx, h, tb, P.d_blkf, P.d_blk, window, sc, P.d_partial, P.max_blocks, P.d_out, stream, P.mode, slow_q);
  else if (R == 4) rc = launch_scan<4>(ctx, h, tb, P.d_blkf, P.d_blk, window, sc, P.d_partial, P.max_blocks, P.d_out, stream, P.mode, slow_q);
  else rc = set_error(GP_INVALID, "train sets spanning more than 4 gpu types are not supported");
  if (!rc && timing) GP_CUDA(cudaEventRecord(ctx->ev[2], stream));
  return rc;
}

// Rank boundaries splitting a train set's space into n_shards contiguous ranges of equal
// layout count (bench.py / multi-GPU fan-out; every range scans with the same kernels).
int train_shard_bounds(gp_ctx* ctx, const int32_t* ids, int n, const gp_train_opts* o, int n_shards,
                       int64_t* bounds) {
  int64_t total = 0;
  int rc = train_space(ctx, ids, n, o, &total);
  if (rc) return rc;
  if (n_shards < 1) return set_error(GP_INVALID, "n_shards must be >= 1");
  for (int i = 0; i <= n_shards; ++i) bounds[i] = (int64_t)((__int128)total * i / n_shards);
  return GP_OK;
}

static void fill_result(PreparedTrain& P, const TrainOut* ho, gp_train_result* out, int32_t* stage_devices) {
  std::memset(out, 0, sizeof *out);
  out->layouts = P.hi - P.lo;
  P.nm[0] = kInfBits;
  P.nm[1] = P.nm[2] = P.nm[3] = LLONG_MAX;
  if (!ho) return;
  P.nm[0] = ho->nm_b0;
  for (int i = 0; i < 3; ++i) P.nm[1 + i] = ho->nm_rank[i];
  out->feasible = ho->best.feasible;
  if (ho->best.rank != LLONG_MAX) {
    out->found = 1;
    out->cost = ho->best.cost;
    out->rank = ho->best.rank;
    out->n_stages = ho->n_stages;
    for (int s = 0; s < ho->n_stages; ++s) {
      out->stage[s].first = ho->first[s];
      out->stage[s].count = ho->count[s];
      out->stage[s].tp = ho->tp[s];
      out->stage[s].dp = ho->dp[s];
      out->stage[s].layers = ho->layers[s];
    }
    if (stage_devices) std::memcpy(stage_devices, P.h.ordered.data(), sizeof(int32_t) * P.h.sp.n);
  }
}

int train_prepare(gp_ctx* ctx, const int32_t* ids, int n, const gp_train_opts* o, int mode) {
  if (!prepared(ctx)) prepared(ctx) = new PreparedTrain();
  PreparedTrain& P = *prepared(ctx);
  GP_CUDA(cudaStreamSynchronize(ctx->stream));  // staging buffer / scratch may be reused
  P.launched = false;
  P.mode = mode;
  P.h = HostSpace();
  int rc = build_space(ctx, ids, n, o, P.h);
  if (rc) return rc;
  P.L = ctx->sc.L;
  P.max_blocks = ctx->num_sms * 8;
  const size_t ib = input_bytes(P.h), tbytes = table_bytes(P.h, P.L, P.max_blocks);
  char* base = static_cast<char*>(ctx_scratch(ctx, ib + tbytes + sizeof(TrainOut) + 512, kArenaTrain));
  if (!base) return GP_CUDA_ERROR;
  char* hp = static_cast<char*>(ctx_pinned(ctx, std::max(ib, sizeof(TrainOut)) + 256));
  if (!hp) return GP_CUDA_ERROR;
  char* in = base;
  char* tab = base + ib;
  carve_prepared(P, in, tab, base, hp);
  P.d_out = carve<TrainOut>(tab, 1);
  const size_t in_bytes = (size_t)(in - base);
  GP_CUDA(cudaMemcpyAsync(base, hp, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += (long long)in_bytes;
  ctx->sum_stages = sum_stages(P.h);
  return GP_OK;
}

// Test hook (gp_debug_layout_costs): per_step of every layout of ranks [lo, hi) as the scan
// kernels compute it (DUMP instantiations of the same code), +inf for memory-infeasible
// layouts. path 0: the whole-space scan a search runs (K1-fast with its best inner run when
// eligible), values of [lo, hi) kept; 1: generic K1 over [lo, hi); 2: K1-fast over [lo, hi)
// with every candidate deferred to k1_deferred; 3: K1-fast over [lo, hi) as a range search
// scans it. *fast_used: K1-fast scored them; *inner: its inner run (-1: generic).
int train_layout_costs(gp_ctx* ctx, const int32_t* ids, int n, const gp_train_opts* o, long long lo,
                       long long hi, int path, double* out, int* fast_used, int* inner) {
  int rc = train_prepare(ctx, ids, n, o, 0);
  if (rc) return rc;
  PreparedTrain& P = *prepared(ctx);
  if (lo < 0 || hi > P.h.total || lo > hi) return set_error(GP_INVALID, "rank range outside the layout space");
  if (hi - lo > (1LL << 26)) return set_error(GP_INVALID, "at most 2^26 ranks per call");
  if (hi == lo) return GP_OK;
  double* d = static_cast<double*>(ctx_scratch(ctx, sizeof(double) * (size_t)(hi - lo), kArenaMisc));
  if (!d) return GP_CUDA_ERROR;
  GP_CUDA(cudaMemsetAsync(d, 0xff, sizeof(double) * (size_t)(hi - lo), ctx->stream));  // NaN: unwritten
  bool fast = false;
  const long long slo = path == 0 ? 0 : lo, shi = path == 0 ? P.h.total : hi;
  rc = launch_prepared(ctx, P, 1, slo, shi, ctx->stream, false, path == 1, -1, d, &fast, path == 2, lo, hi);
  if (rc) return rc;
  if (inner) *inner = fast ? P.h.sp.R - 1 : -1;  // K1-fast scans the last type run innermost
  TrainOut* ho = reinterpret_cast<TrainOut*>(ctx_pinned(ctx, sizeof(TrainOut)));
  GP_CUDA(cudaMemcpyAsync(ho, P.d_out, sizeof(TrainOut), cudaMemcpyDeviceToHost, ctx->stream));
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ho->overflow) return set_error(GP_INVALID, "deferred queue overflow: use a smaller range");
  GP_CUDA(cudaMemcpy(out, d, sizeof(double) * (size_t)(hi - lo), cudaMemcpyDeviceToHost));
  if (fast_used) *fast_used = fast;
  return GP_OK;
}

int train_launch(gp_ctx* ctx, int window, long long lo, long long hi) {
  PreparedTrain* PP = prepared(ctx);
  if (!PP) return set_error(GP_INVALID, "gp_train_launch without gp_train_prepare");
  return launch_prepared(ctx, *PP, window, lo, hi, ctx->stream, ctx->timing);
}

int train_collect(gp_ctx* ctx, gp_train_result* out, int32_t* stage_devices) {
  std::memset(out, 0, sizeof *out);
  PreparedTrain* PP = prepared(ctx);
  if (!PP || !PP->launched) return set_error(GP_INVALID, "gp_train_collect without gp_train_launch");
  PreparedTrain& P = *PP;
  if (P.h.total == 0 || P.lo == P.hi) {
    GP_CUDA(cudaStreamSynchronize(ctx->stream));
    fill_result(P, nullptr, out, stage_devices);
    return GP_OK;
  }
  TrainOut* ho = reinterpret_cast<TrainOut*>(ctx_pinned(ctx, sizeof(TrainOut)));
  GP_CUDA(cudaMemcpyAsync(ho, P.d_out, sizeof(TrainOut), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->d2h_bytes += (long long)sizeof(TrainOut);
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (ho->overflow) {  // too many deferred candidates: rescan the range with the generic K1
    int rc = launch_prepared(ctx, P, P.window, P.lo, P.hi, ctx->stream, false, true);
    if (rc) return rc;
    GP_CUDA(cudaMemcpyAsync(ho, P.d_out, sizeof(TrainOut), cudaMemcpyDeviceToHost, ctx->stream));
    GP_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  fill_result(P, ho, out, stage_devices);
  g_memo_stats.poll();
  return GP_OK;
}

void train_last_nm(gp_ctx* ctx, long long nm[4]) {
  PreparedTrain* PP = prepared(ctx);
  for (int i = 0; i < 4; ++i) nm[i] = PP ? PP->nm[i] : (i ? LLONG_MAX : kInfBits);
}

// ---- window-independent memo of constrained_search (see NearMin). A full-range search
// of a train set is stored with its near-minimum summary and the decoded plan of the rank
// that won; a later call with another window derives its winner from the summary exactly
// and is answered from the memo when that winner is the stored plan (always, unless a
// two-ulp near tie resolves differently under the new window — then it is re-scanned).
struct TrainMemoEntry {
  gp_train_result res;
  std::vector<int32_t> ordered;
  NearMin nm;  // keys = ranks (rank order == key order)
};
struct TrainMemo {
  std::unordered_map<std::string, TrainMemoEntry> map;
};
constexpr size_t kMemoCap = 1 << 16;


// host merge of two NearMin summaries held as {b0, rank0, rank1, rank2}
void train_nm_merge(long long a[4], const long long b[4]) {
  NearMin x{a[0], {a[1], a[2], a[3]}, 0}, y{b[0], {b[1], b[2], b[3]}, 0};
  nm_merge(x, y);
  a[0] = x.b0;
  for (int i = 0; i < 3; ++i) a[1 + i] = x.key[i];
}

void train_memo_free(gp_ctx* ctx) {
  delete static_cast<TrainMemo*>(ctx->train_memo);
  ctx->train_memo = nullptr;
}

std::string train_memo_key(const int32_t* ids, int n, const gp_train_opts* o, int mode) {
  std::vector<int32_t> v(ids, ids + n);
  std::sort(v.begin(), v.end());  // the search canonicalises the order itself
  v.push_back(o->max_stages_per_type);
  v.push_back(o->device_granularity_limit);
  v.push_back(mode);
  return std::string(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(int32_t));
}

void train_memo_put(gp_ctx* ctx, const std::string& key, const gp_train_result& r, const int32_t* ordered,
                    int n, const long long nm[4]);

// stores a search just collected on ctx (the plan's device order is the prepared set's)
void train_memo_put_last(gp_ctx* ctx, const std::string& key, const gp_train_result& r, const long long nm[4]) {
  PreparedTrain* PP = prepared(ctx);
  if (!PP) return;
  train_memo_put(ctx, key, r, PP->h.ordered.data(), PP->h.sp.n, nm);
}

bool train_memo_get(gp_ctx* ctx, const std::string& key, int window, gp_train_result* out,
                    int32_t* stage_devices) {
  if (!ctx->memo || !ctx->train_memo) return false;
  auto& map = static_cast<TrainMemo*>(ctx->train_memo)->map;
  auto it = map.find(key);
  if (it == map.end()) return false;
  const TrainMemoEntry& e = it->second;
  double cost;
  const long long rank = nm_winner(e.nm, window, cost);
  if (rank != (e.res.found ? e.res.rank : LLONG_MAX)) return false;
  *out = e.res;
  g_memo_stats.hits++;
  if (out->found) {
    out->cost = cost;
    if (stage_devices) std::memcpy(stage_devices, e.ordered.data(), sizeof(int32_t) * e.ordered.size());
  }
  return true;
}

void train_memo_put(gp_ctx* ctx, const std::string& key, const gp_train_result& r, const int32_t* ordered,
                    int n, const long long nm[4]) {
  if (!ctx->memo) return;
  if (!ctx->train_memo) ctx->train_memo = new TrainMemo();
  auto& map = static_cast<TrainMemo*>(ctx->train_memo)->map;
  if (map.size() >= kMemoCap) map.clear();
  TrainMemoEntry& e = map[key];
  e.res = r;
  if (r.found) e.ordered.assign(ordered, ordered + n);
  e.nm.b0 = nm[0];
  for (int i = 0; i < 3; ++i) e.nm.key[i] = nm[1 + i];
  e.nm.feasible = r.feasible;
}

int train_search(gp_ctx* ctx, const int32_t* ids, int n, int window, const gp_train_opts* o,
                 long long lo, long long hi, gp_train_result* out, int32_t* stage_devices, int mode) {
  std::memset(out, 0, sizeof *out);
  int rc = train_prepare(ctx, ids, n, o, mode);
  if (!rc) rc = train_launch(ctx, window, lo, hi);
  if (!rc) rc = train_collect(ctx, out, stage_devices);
  return rc;
}

// fn(i) for i < n on up to max_threads host threads (inline below 64 items)
template <typename F>
static void parallel_sets(int n, int max_threads, F fn) {
  const int nt = std::min(max_threads, n / 32);
  if (nt <= 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (int i = t; i < n; i += nt) fn(i);
    });
  for (auto& x : th) x.join();
}

// Batched constrained_search over many train sets (the scheduler's evaluation batches):
// every set's inputs travel in ONE H2D copy, all tables + scans are enqueued back to back,
// the results come back in ONE D2H copy with ONE synchronisation.
// Scans every set on ctx (no memo): one H2D, all launches on the lane streams, one D2H.
// Returns per set the NearMin summary and the canonical device order for the memo.
static int train_batch_run(gp_ctx* ctx, int n_sets, const int32_t* const* ids, const int32_t* ns, int window,
                           const gp_train_opts* o, gp_train_result* outs, int32_t* const* stage_devices,
                           int mode, std::vector<std::array<long long, 4>>& nms,
                           std::vector<std::vector<int32_t>>& ordered, int host_threads) {
  nms.assign(n_sets, {});
  ordered.assign(n_sets, {});
  if (n_sets <= 0) return GP_OK;
  auto tick = std::chrono::steady_clock::now();
  auto lap = [&](int k) {
    const auto t = std::chrono::steady_clock::now();
    g_memo_stats.ph[k] += std::chrono::duration<double>(t - tick).count();
    tick = t;
  };
  std::vector<PreparedTrain> Ps(n_sets);
  std::vector<size_t> in_at(n_sets + 1, 0), tab_at(n_sets + 1, 0);  // per-set carve offsets
  {  // host enumeration of every set's space, on several host threads for large batches
    std::vector<int> rcs(n_sets, GP_OK);
    std::vector<std::string> errs(n_sets);
    parallel_sets(n_sets, host_threads, [&](int i) {
      rcs[i] = build_space(ctx, ids[i], ns[i], o, Ps[i].h);
      if (rcs[i]) {
        errs[i] = gp_last_error();  // (the message is thread-local)
        return;
      }
      Ps[i].mode = mode;
      Ps[i].L = ctx->sc.L;
      Ps[i].max_blocks = std::min(ctx->num_sms * 8, (int)std::max<long long>(1, Ps[i].h.total / 4096));
    });
    for (int i = 0; i < n_sets; ++i)
      if (rcs[i]) return set_error(rcs[i], errs[i]);
  }
  for (int i = 0; i < n_sets; ++i) {
    in_at[i + 1] = in_at[i] + input_bytes(Ps[i].h);
    tab_at[i + 1] = tab_at[i] + table_bytes(Ps[i].h, Ps[i].L, Ps[i].max_blocks);
  }
  const size_t ib = in_at[n_sets], tbytes = tab_at[n_sets];
  const size_t out_bytes = sizeof(TrainOut) * n_sets;
  lap(0);
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  char* base = static_cast<char*>(ctx_scratch(ctx, ib + tbytes + out_bytes + 1024, kArenaTrain));
  if (!base) return GP_CUDA_ERROR;
  char* hp = static_cast<char*>(ctx_pinned(ctx, std::max(ib, out_bytes) + 1024));
  if (!hp) return GP_CUDA_ERROR;
  // (input_bytes / table_bytes bound what carve_prepared takes: the sets carve in parallel)
  parallel_sets(n_sets, host_threads, [&](int i) {
    char* in_i = base + in_at[i];
    char* tab_i = base + ib + tab_at[i];
    carve_prepared(Ps[i], in_i, tab_i, base, hp);
  });
  char* tab = base + ib + tbytes;
  TrainOut* d_out = carve<TrainOut>(tab, n_sets);
  for (int i = 0; i < n_sets; ++i) Ps[i].d_out = d_out + i;
  const size_t in_bytes = ib;
  GP_CUDA(cudaMemcpyAsync(base, hp, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += (long long)in_bytes;
  lap(1);
  // the sets run on kTrainLanes streams so that small sets overlap on the GPU
  constexpr int NL = gp_ctx::kTrainLanes;
  if (!ctx->lane[0]) {
    for (int l = 0; l < NL; ++l) GP_CUDA(cudaStreamCreateWithFlags(&ctx->lane[l], cudaStreamNonBlocking));
    for (int l = 0; l <= NL; ++l) GP_CUDA(cudaEventCreateWithFlags(&ctx->ev_lane[l], cudaEventDisableTiming));
  }
  GP_CUDA(cudaEventRecord(ctx->ev_lane[NL], ctx->stream));  // inputs are on the device
  for (int l = 0; l < NL; ++l) GP_CUDA(cudaStreamWaitEvent(ctx->lane[l], ctx->ev_lane[NL], 0));
  // small spaces: the fused one-CTA-per-set kernel, one launch per type-run count
  std::vector<int> small_of[GP_MAX_TYPES + 1];
  for (int i = 0; i < n_sets; ++i) {
    const HostSpace& h = Ps[i].h;
    if (h.total > 0 && h.total <= kSmallLayouts && h.sp.R >= 1 && h.sp.R <= 4) small_of[h.sp.R].push_back(i);
  }
  std::vector<char> is_small(n_sets, 0);
  for (int R = 1; R <= 4; ++R) {
    const int ns_ = (int)small_of[R].size();
    if (ns_ == 0) continue;
    std::vector<SmallSet> ss(ns_);
    for (int j = 0; j < ns_; ++j) {
      PreparedTrain& P = Ps[small_of[R][j]];
      is_small[small_of[R][j]] = 1;
      P.lo = 0;
      P.hi = P.h.total;
      P.window = window;
      P.launched = true;
      SmallSet& S = ss[j];
      S.sp = P.h.sp;
      S.tb = prepared_tables(ctx, P);
      ScanRange rg{};
      rank_split(P.h, 0, rg.p_lo, rg.s_lo);
      rank_split(P.h, P.h.total, rg.p_hi, rg.s_hi);
      rg.n_pref = rg.p_hi - rg.p_lo + (rg.s_hi > 0 ? 1 : 0);
      rg.chunk = std::max(1LL, rg.n_pref / (2 * (kK1Threads / 32)));
      S.rg = rg;
      S.meta = P.d_meta;
      S.run_start = P.d_run_start;
      S.items = P.d_items;
      S.choices = P.d_choices;
      S.blk = P.d_blk;
      S.blkf = P.d_blkf;
      S.stage = P.d_stage;
      S.opt = P.d_opt;
      S.tin = P.d_tin;
      S.tx = P.d_tx;
      S.fd = P.d_fd;
      S.suf = P.d_suf;
      S.partial = P.d_partial;
      S.out = P.d_out;
      S.nblk = P.h.nblk;
      S.n_items = (int)P.h.items.size();
      S.n_choices = (int)P.h.choices.size();
      S.mode = P.mode;
    }
    SmallSet* d_ss = nullptr;  // descriptors: stream-ordered allocation, freed after the launch
    GP_CUDA(cudaMallocAsync(&d_ss, sizeof(SmallSet) * ns_, ctx->lane[R % NL]));
    GP_CUDA(cudaMemcpyAsync(d_ss, ss.data(), sizeof(SmallSet) * ns_, cudaMemcpyHostToDevice, ctx->lane[R % NL]));
    ctx->h2d_bytes += (long long)(sizeof(SmallSet) * ns_);
    const double numer = ctx->sc.tokens > 0 ? ctx->sc.act_tok_h2 : 0.0;
    auto launch = [&](auto kern) {
      kern<<<ns_, kK1Threads, 0, ctx->lane[R % NL]>>>(d_ss, ctx->sc, ctx->d_type, ctx->d_machine, ctx->d_flops,
                                                      ctx->d_hbm_cap, ctx->d_links, ctx->N, ctx->d_ceff, numer,
                                                      window);
    };
    if (R == 1) launch(k_train_small<1>);
    else if (R == 2) launch(k_train_small<2>);
    else if (R == 3) launch(k_train_small<3>);
    else launch(k_train_small<4>);
    ctx->launches++;
    GP_CUDA(cudaGetLastError());
    GP_CUDA(cudaFreeAsync(d_ss, ctx->lane[R % NL]));  // (a pageable-source copy is staged on return)
  }
  // (measured: sending the sets that fill the GPU alone to one lane, the rest round-robin on
  // the others, is no faster on the C5 schedule)
  for (int i = 0, k = 0; i < n_sets; ++i) {
    if (is_small[i]) continue;
    const int l = k++ % NL;
    int rc = launch_prepared(ctx, Ps[i], window, 0, -1, ctx->lane[l], false, false, l);
    if (rc) return rc;
  }
  for (int l = 0; l < NL; ++l) {
    GP_CUDA(cudaEventRecord(ctx->ev_lane[l], ctx->lane[l]));
    GP_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_lane[l], 0));
  }
  TrainOut* ho = reinterpret_cast<TrainOut*>(hp);
  GP_CUDA(cudaMemcpyAsync(ho, d_out, out_bytes, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->d2h_bytes += (long long)out_bytes;
  lap(2);
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  lap(3);
  for (int i = 0; i < n_sets; ++i) {
    if (Ps[i].h.total > 0 && ho[i].overflow) {  // rescan with the generic K1
      int rc = launch_prepared(ctx, Ps[i], window, 0, -1, ctx->stream, false, true);
      if (rc) return rc;
      GP_CUDA(cudaMemcpyAsync(ho + i, d_out + i, sizeof(TrainOut), cudaMemcpyDeviceToHost, ctx->stream));
      GP_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  }
  for (int i = 0; i < n_sets; ++i) {
    const bool ran = Ps[i].h.total > 0;
    fill_result(Ps[i], ran ? ho + i : nullptr, outs + i, stage_devices ? stage_devices[i] : nullptr);
    for (int k = 0; k < 4; ++k) nms[i][k] = Ps[i].nm[k];
    ordered[i] = Ps[i].h.ordered;
    g_memo_stats.scans++;
    g_memo_stats.layouts += Ps[i].h.total;
    {
      int b = 0;
      for (long long t = Ps[i].h.total; t >= 10 && b < 11; t /= 10) ++b;
      g_memo_stats.size_sets[b]++;
      g_memo_stats.size_layouts[b] += Ps[i].h.total;
    }
  }
  lap(4);
  g_memo_stats.poll();
  return GP_OK;
}

// Batched constrained_search over many train sets (the scheduler's evaluation batches):
// memo hits are answered on the host; the rest is scanned by train_batch_run — split over
// the context's devices (gp_ctx_create_multi) by layout count when it has peers.
int train_batch(gp_ctx* ctx, int n_sets, const int32_t* const* ids, const int32_t* ns, int window,
                const gp_train_opts* o, gp_train_result* outs, int32_t* const* stage_devices, int mode) {
  if (n_sets <= 0) return GP_OK;
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  std::vector<std::string> keys(n_sets);
  parallel_sets(n_sets, std::min(16, hw), [&](int i) { keys[i] = train_memo_key(ids[i], ns[i], o, mode); });
  std::vector<int> todo;
  for (int i = 0; i < n_sets; ++i)
    if (!train_memo_get(ctx, keys[i], window, outs + i, stage_devices ? stage_devices[i] : nullptr))
      todo.push_back(i);
  if (todo.empty()) return GP_OK;
  const int q = (int)todo.size();
  std::vector<std::array<long long, 4>> nms(q);
  std::vector<std::vector<int32_t>> ordered(q);
  std::vector<gp_train_result> res(q);
  std::vector<int> dev_of(q, 0);
  const int D = 1 + (int)ctx->peers.size();
  if (D > 1 && q > 1) {  // longest-processing-time assignment by layout count
    std::vector<std::pair<long long, int>> sz(q);
    std::vector<int> src(q, GP_OK);
    std::vector<std::string> serr(q);
    parallel_sets(q, std::min(16, hw), [&](int j) {
      int64_t total = 0;
      src[j] = train_space(ctx, ids[todo[j]], ns[todo[j]], o, &total);
      if (src[j]) serr[j] = gp_last_error();  // (thread-local)
      sz[j] = {(long long)total, j};
    });
    for (int j = 0; j < q; ++j)
      if (src[j]) return set_error(src[j], serr[j]);
    std::sort(sz.begin(), sz.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
    long long all = 0;
    for (const auto& e : sz) all += e.first;
    // a batch worth well under a millisecond of scanning stays on one device: the per-device
    // threads, uploads and synchronisations would cost more than they save
    if (all >= kBatchSplitMinLayouts) {
      std::vector<long long> load(D, 0);
      for (const auto& e : sz) {
        const int d = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        dev_of[e.second] = d;
        load[d] += e.first + 100000;  // + per-set fixed cost
      }
    }
  }
  std::vector<int> rcs(D, GP_OK);
  std::vector<std::string> errs(D);
  std::vector<std::vector<int>> part(D);
  for (int j = 0; j < q; ++j) part[dev_of[j]].push_back(j);
  int busy = 0;  // device threads of this batch share the host's cores for set preparation
  for (int d = 0; d < D; ++d) busy += part[d].empty() ? 0 : 1;
  const int host_threads = std::max(1, std::min(16, hw / std::max(1, busy)));
  auto run = [&](int d) {
    gp_ctx* c = d == 0 ? ctx : ctx->peers[d - 1];
    const std::vector<int>& pj = part[d];
    if (pj.empty()) return;
    cudaSetDevice(c->device);
    std::vector<const int32_t*> id2;
    std::vector<int32_t> n2;
    std::vector<int32_t*> sd2;
    for (int j : pj) {
      id2.push_back(ids[todo[j]]);
      n2.push_back(ns[todo[j]]);
      sd2.push_back(stage_devices ? stage_devices[todo[j]] : nullptr);
    }
    std::vector<gp_train_result> r2(pj.size());
    std::vector<std::array<long long, 4>> nm2;
    std::vector<std::vector<int32_t>> or2;
    rcs[d] = train_batch_run(c, (int)pj.size(), id2.data(), n2.data(), window, o, r2.data(),
                             stage_devices ? sd2.data() : nullptr, mode, nm2, or2, host_threads);
    if (rcs[d]) {
      errs[d] = gp_last_error();
      return;
    }
    for (size_t k = 0; k < pj.size(); ++k) {
      res[pj[k]] = r2[k];
      nms[pj[k]] = nm2[k];
      ordered[pj[k]] = std::move(or2[k]);
    }
  };
  if (D == 1 || q == 1) {
    run(0);
  } else {
    std::vector<std::thread> th;
    for (int d = 1; d < D; ++d) th.emplace_back(run, d);
    run(0);
    for (auto& t : th) t.join();
    cudaSetDevice(ctx->device);
  }
  for (int d = 0; d < D; ++d)
    if (rcs[d]) return set_error(rcs[d], errs[d].empty() ? std::string("train batch failed") : errs[d]);
  for (int j = 0; j < q; ++j) {
    outs[todo[j]] = res[j];
    train_memo_put(ctx, keys[todo[j]], res[j], ordered[j].data(), (int)ordered[j].size(), nms[j].data());
  }
  return GP_OK;
}

}  // namespace gp
