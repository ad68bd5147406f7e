// partition.cu — sm_100a kernels for the repartition solver:
//   graph_partition_candidates (src/partition.cpp:369-406) with build_units
//   (:37-80), State (:83-163), TopK (:174-210), exact_enumeration (:212-222),
//   greedy_seed (:224-269), local_search (:271-350), compute_fraction (:360-367).
//
// K5a units      unit folds (flops, hbm, internal link, cross matrix) — one CTA per unit row
// K5b exact      one thread per bisection mask (n <= exact_threshold)
// K5c restarts   one thread-block cluster per restart (1..8 CTAs, as many as fill the
//                GPU): SplitMix64-perturbed order (counter-based, parallel), CTA-wide
//                stable sort, greedy seed, then the whole steepest-ascent loop on chip:
//                every step scores all moves and all (train, rollout) swaps in parallel
//                — the cluster's CTAs hold identical replicated state and each scores its
//                share of the rows — and reduces lexicographically on (gain desc, scan
//                position asc), the reference's first strict max, through distributed
//                shared memory (one cluster barrier per step).
// K5d topk       one thread replays TopK::offer in the reference's offer order.
// Objective/fraction divisions by the fixed totals use a correctly rounded
// reciprocal with one FMA residual correction (Markstein), identical to IEEE
// division for these operands; every other fp operation keeps reference order.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "gp_internal.h"

namespace gp {

constexpr int kMaxUnits = 4096;
constexpr int kK5Threads = 1024;

struct Units {
  int n;
  const double* flops;
  const double* hbm;
  const double* internal;
  const double* cross;  // n x n
  const int* mem_off;   // members of unit i: mem_ids[mem_off[i] .. mem_off[i+1])
  const int* mem_ids;
};

struct Totals {
  double flops, hbm, link;
  double y_flops, y_hbm, y_link;  // RN(1/total)
};

__device__ __forceinline__ double div_rn_recip2(double a, double b, double y) {
  const double q = __dmul_rn(a, y);
  const double r = __fma_rn(-q, b, a);
  return __fma_rn(r, y, q);
}

// ---------------------------------------------------------------- K5a units
__global__ void k5_units(int n, const int* __restrict__ mem_off, const int* __restrict__ mem_ids,
                         const double* __restrict__ dflops, const double* __restrict__ dhbm,
                         const double* __restrict__ links, int N, double* __restrict__ uflops,
                         double* __restrict__ uhbm, double* __restrict__ uint_,
                         double* __restrict__ cross) {
  const int i = blockIdx.x;
  const int* mi = mem_ids + mem_off[i];
  const int ni = mem_off[i + 1] - mem_off[i];
  if (threadIdx.x == 0) {
    double f = 0, h = 0, in = 0;
    for (int a = 0; a < ni; ++a) {
      f += dflops[mi[a]];
      h += dhbm[mi[a]];
      for (int b = a + 1; b < ni; ++b) in += links[(size_t)mi[a] * N + mi[b]];
    }
    uflops[i] = f;
    uhbm[i] = h;
    uint_[i] = in;
    cross[(size_t)i * n + i] = 0;
  }
  for (int j = i + 1 + threadIdx.x; j < n; j += blockDim.x) {
    const int* mj = mem_ids + mem_off[j];
    const int nj = mem_off[j + 1] - mem_off[j];
    double bw = 0;
    for (int a = 0; a < ni; ++a)
      for (int b = 0; b < nj; ++b) bw += links[(size_t)mi[a] * N + mj[b]];
    cross[(size_t)i * n + j] = bw;
    cross[(size_t)j * n + i] = bw;
  }
}

// totals: sequential folds in unit order (src/partition.cpp:75-79)
// The total-link fold is inherently sequential (fp order); the CTA streams each row of
// the cross matrix into shared memory (double-buffered) so the folding thread only
// waits on DADD latency, not on L2.
__global__ void k5_totals(Units u, Totals* __restrict__ tot, double* __restrict__ base_score) {
  constexpr int kChunk = 2048;
  __shared__ double row[2][kChunk];
  double tl = 0;
  int buf = 0;
  for (int i = 0; i < u.n; ++i) {
    if (threadIdx.x == 0) tl += u.internal[i];
    for (int c0 = i + 1; c0 < u.n; c0 += kChunk) {
      const int c1 = min(u.n, c0 + kChunk);
      for (int j = c0 + threadIdx.x; j < c1; j += blockDim.x) row[buf][j - c0] = u.cross[(size_t)i * u.n + j];
      __syncthreads();
      if (threadIdx.x == 0)
        for (int j = 0; j < c1 - c0; ++j) tl += row[buf][j];
      buf ^= 1;  // the next chunk fills the other buffer while thread 0 folds this one
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tf = 0.0, th = 0.0;
    for (int i = 0; i < u.n; ++i) tf += u.flops[i];
    for (int i = 0; i < u.n; ++i) th += u.hbm[i];
    tot->flops = tf;
    tot->hbm = th;
    tot->link = tl;
    tot->y_flops = 1.0 / tf;
    tot->y_hbm = 1.0 / th;
    tot->y_link = tl > 0 ? 1.0 / tl : 0.0;
  }
  __syncthreads();
  // local_search base score (src/partition.cpp:273-282): per unit, fold over j != i
  for (int i = threadIdx.x; i < u.n; i += blockDim.x) {
    double d = 0;
    for (int j = 0; j < u.n; ++j)
      if (j != i) d += u.cross[(size_t)i * u.n + j];
    d += 2.0 * u.internal[i];
    if (u.n > 1) d /= static_cast<double>(u.n - 1);
    base_score[i] = d * u.flops[i];
  }
}

// ---------------------------------------------------------------- K5b exact
struct Offer {
  double obj;
  int valid;
  int pad;
};

__global__ void k5_exact(Units u, const Totals* __restrict__ tot, double lo, double hi,
                         Offer* __restrict__ offers) {
  const unsigned long long mask = 1ull + (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int n = u.n;
  if (mask + 1 >= (1ull << n)) return;
  double ltt[20];
  for (int j = 0; j < n; ++j) ltt[j] = 0;
  double link_train = 0, hbm_train = 0, flops_train = 0;
  for (int i = 0; i < n; ++i) {
    if (!(mask & (1ull << i))) continue;
    link_train += ltt[i] + u.internal[i];  // State::add
    hbm_train += u.hbm[i];
    flops_train += u.flops[i];
    for (int j = 0; j < n; ++j)
      if (j != i) ltt[j] += u.cross[(size_t)i * n + j];
  }
  const Totals T = *tot;
  const double f = flops_train / T.flops;
  Offer o;
  o.valid = f >= lo && f <= hi;
  const double lf = T.link > 0 ? link_train / T.link : 0;
  o.obj = lf + (T.hbm - hbm_train) / T.hbm;
  o.pad = 0;
  offers[mask - 1] = o;
}

// ---------------------------------------------------------------- K5c restarts
struct RestartOut {
  double obj;
  int ok;
  int count;
  unsigned long long steps;
};

__device__ __forceinline__ unsigned long long smx(unsigned long long x) {
  unsigned long long z = x;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

struct Cand {
  double gain;
  int pos;  // scan position: moves i, swaps n + a*n + b
};

__device__ __forceinline__ bool cand_better(const Cand& x, const Cand& y) {
  return x.gain > y.gain || (x.gain == y.gain && x.pos < y.pos);
}

__device__ Cand block_best(Cand c, Cand* sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand d;
    d.gain = __shfl_xor_sync(0xffffffffu, c.gain, o);
    d.pos = __shfl_xor_sync(0xffffffffu, c.pos, o);
    if (cand_better(d, c)) c = d;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sm[wid] = c;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  c = lane < nw ? sm[lane] : Cand{-1e300, INT_MAX};
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand d;
    d.gain = __shfl_xor_sync(0xffffffffu, c.gain, o);
    d.pos = __shfl_xor_sync(0xffffffffu, c.pos, o);
    if (cand_better(d, c)) c = d;
  }
  return c;
}

struct SState {
  double link_train, hbm_train, flops_train;
  int count;
  int pick;
  int flag;
  int n_tr, n_ro;
};

// One cluster of csize CTAs per (band, restart): blockIdx.x / csize = band * restarts + r (a
// scheduler iteration's bands run in one launch); band b's limits are bands[b] = (lo, hi).
// Every CTA of a cluster runs the same seed and applies the same steps (replicated state);
// the step scan is split by CTA rank and the winner is the lexicographic best of the CTAs'
// winners, so the result is independent of csize (csize == 1: no cluster operations).
__global__ void __launch_bounds__(kK5Threads) k5_restart(Units u, const Totals* __restrict__ tot,
                                                         const double* __restrict__ base_score,
                                                         const double2* __restrict__ bands, int restarts,
                                                         unsigned long long seed,
                                                         unsigned char* __restrict__ in_train_out,
                                                         RestartOut* __restrict__ out, int csize) {
  extern __shared__ unsigned char smem[];
  const int n = u.n;
  double* ltt = reinterpret_cast<double*>(smem);
  double* key = ltt + n;                       // perturbed scores, then reused
  int* order = reinterpret_cast<int*>(key + n);
  int* tr = order + n;                         // train unit list (ascending)
  int* ro = tr + n;                            // rollout unit list (ascending)
  double* uf = reinterpret_cast<double*>(ro + n + (n & 1));  // unit flops / hbm / internal (smem copies)
  double* uh = uf + n;
  double* ui = uh + n;
  unsigned char* in_tr = reinterpret_cast<unsigned char*>(ui + n);
  __shared__ SState S;
  __shared__ Cand red[32];
  __shared__ int ired[32];
  __shared__ Cand cbest[2];  // this CTA's step winner (by step parity), read by the cluster
  __shared__ int lc_t[32], lc_r[32];
  const int crank = blockIdx.x % csize, rid = blockIdx.x / csize;
  const int r = rid % restarts;
  const double lo = bands[rid / restarts].x, hi = bands[rid / restarts].y;
  const Totals T = *tot;
  const int tid = threadIdx.x, nth = blockDim.x;

  // ---- perturbed order: score_i *= 0.5 + U_i (SplitMix64 stream of this restart)
  const unsigned long long s0 = seed + (unsigned long long)r * 0x9e3779b97f4a7c15ull;
  for (int i = tid; i < n; i += nth) {
    double sc = base_score[i];
    if (r > 0) {
      const unsigned long long z = smx(s0 + (unsigned long long)(i + 1) * 0x9e3779b97f4a7c15ull);
      sc *= 0.5 + static_cast<double>(z >> 11) * 0x1.0p-53;
    }
    key[i] = sc;
    ltt[i] = 0;
    in_tr[i] = 0;
    uf[i] = u.flops[i];
    uh[i] = u.hbm[i];
    ui[i] = u.internal[i];
  }
  __syncthreads();
  // stable sort by score desc: rank_i = #{score_j > score_i} + #{j < i : score_j == score_i}
  for (int i = tid; i < n; i += nth) {
    const double si = key[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double sj = key[j];
      rank += (sj > si) || (sj == si && j < i);
    }
    order[rank] = i;
  }
  if (tid == 0) {
    S.link_train = S.hbm_train = S.flops_train = 0;
    S.count = 0;
  }
  __syncthreads();
  const double bhi = (1.0 < hi) ? 1.0 : hi;
  const double blo = (lo < 0.0) ? 0.0 : lo;
  const double target = blo + (r + 0.5) / restarts * (bhi - blo);

  auto frac = [&](double ft) { return div_rn_recip2(ft, T.flops, T.y_flops); };
  auto in_band = [&](double f) { return f >= lo && f <= hi; };
  // State::add / State::remove with the parallel link_to_train update
  auto add = [&](int i) {
    __syncthreads();
    if (tid == 0) {
      S.link_train += ltt[i] + ui[i];
      S.hbm_train += uh[i];
      S.flops_train += uf[i];
      S.count++;
      in_tr[i] = 1;
    }
    __syncthreads();
    for (int j = tid; j < n; j += nth)
      if (j != i) ltt[j] += u.cross[(size_t)i * n + j];
    __syncthreads();
  };
  auto remove = [&](int i) {
    __syncthreads();
    for (int j = tid; j < n; j += nth)
      if (j != i) ltt[j] -= u.cross[(size_t)i * n + j];
    __syncthreads();
    if (tid == 0) {
      in_tr[i] = 0;
      S.link_train -= ltt[i] + ui[i];
      S.hbm_train -= uh[i];
      S.flops_train -= uf[i];
      S.count--;
    }
    __syncthreads();
  };
  // remove(a) then add(b) in one pass: every element sees the same two roundings in the same
  // order (ltt[j] - cross[a][j], then + cross[b][j]), and the totals the same sequence
  auto swap_units = [&](int a, int b) {
    __syncthreads();
    if (tid == 0) {
      const double la = ltt[a] + ui[a];                                  // remove: ltt[a] is not updated
      const double lb2 = (ltt[b] - u.cross[(size_t)a * n + b]) + ui[b];  // add: ltt[b] after the removal
      S.link_train -= la;
      S.link_train += lb2;
      S.hbm_train -= uh[a];
      S.hbm_train += uh[b];
      S.flops_train -= uf[a];
      S.flops_train += uf[b];
      in_tr[a] = 0;
      in_tr[b] = 1;
    }
    __syncthreads();  // (thread 0 read ltt[a], ltt[b] before the update)
    const double* ca = u.cross + (size_t)a * n;
    const double* cb = u.cross + (size_t)b * n;
    for (int j = tid; j < n; j += nth) {
      double v = ltt[j];
      if (j != a) v -= ca[j];
      if (j != b) v += cb[j];
      ltt[j] = v;
    }
    __syncthreads();
  };
  // argmin of flops over units with in_tr == want (first index on ties); n if none
  auto argmin_flops = [&](int want) {
    double bv = 0;
    int bi = INT_MAX;
    for (int i = tid; i < n; i += nth) {
      if (in_tr[i] != want) continue;
      const double f = uf[i];
      if (bi == INT_MAX || f < bv || (f == bv && i < bi)) {
        bv = f;
        bi = i;
      }
    }
    Cand c{bi == INT_MAX ? -1e300 : -bv, bi};
    c = block_best(c, red);
    return c.pos == INT_MAX ? n : c.pos;
  };

  // ---- greedy_seed (src/partition.cpp:224-269)
  bool ok = true;
  for (int oi = 0; oi < n; ++oi) {
    if (frac(S.flops_train) >= target) break;
    if (S.count + 1 >= n) break;
    add(order[oi]);
  }
  for (int guard = 0; guard < 4 * n; ++guard) {
    const double f = frac(S.flops_train);
    if (in_band(f)) break;
    if (f > hi) {
      if (S.count <= 1) {
        ok = false;
        break;
      }
      const int pick = argmin_flops(1);
      remove(pick);
    } else {
      if (S.count + 1 >= n) {
        ok = false;
        break;
      }
      // first unit in `order` outside train whose move keeps f <= hi + 1e-15
      int best_o = INT_MAX;
      for (int oi = tid; oi < n; oi += nth) {
        const int i = order[oi];
        if (in_tr[i]) continue;
        if (frac(S.flops_train + uf[i]) <= hi + 1e-15) best_o = min(best_o, oi);
      }
      for (int o = 16; o > 0; o >>= 1) best_o = min(best_o, __shfl_xor_sync(0xffffffffu, best_o, o));
      __syncthreads();
      if ((tid & 31) == 0) ired[tid >> 5] = best_o;
      __syncthreads();
      if (tid < 32) {
        int v = tid < (nth >> 5) ? ired[tid] : INT_MAX;
        for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (tid == 0) S.pick = v;
      }
      __syncthreads();
      int pick = S.pick == INT_MAX ? n : order[S.pick];
      if (pick == n) {
        pick = argmin_flops(0);
        if (pick == n) {
          ok = false;
          break;
        }
      }
      add(pick);
    }
  }
  ok = ok && in_band(frac(S.flops_train)) && S.count > 0 && S.count < n;

  // ---- steepest ascent (src/partition.cpp:302-347)
  unsigned long long steps = 0;
  int par = 0;
  while (ok) {
    {  // ascending train / rollout unit lists (scan order of the swap loops): every warp
       // ballots 32 units, a per-round warp prefix places them
      const int l_ = tid & 31, w_ = tid >> 5, nw_ = nth >> 5;
      int bt = 0, br = 0;
      for (int b0 = 0; b0 < n; b0 += nth) {
        const int i = b0 + tid;
        const bool t = i < n && in_tr[i], rr = i < n && !in_tr[i];
        const unsigned mt = __ballot_sync(0xffffffffu, t), mr = __ballot_sync(0xffffffffu, rr);
        if (l_ == 0) {
          lc_t[w_] = __popc(mt);
          lc_r[w_] = __popc(mr);
        }
        __syncthreads();
        int pt = 0, pr = 0, at = 0, ar = 0;  // this warp's exclusive offsets, the round's totals
        if (l_ < nw_) {
          at = lc_t[l_];
          ar = lc_r[l_];
          pt = l_ < w_ ? at : 0;
          pr = l_ < w_ ? ar : 0;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          pt += __shfl_xor_sync(0xffffffffu, pt, o);
          pr += __shfl_xor_sync(0xffffffffu, pr, o);
          at += __shfl_xor_sync(0xffffffffu, at, o);
          ar += __shfl_xor_sync(0xffffffffu, ar, o);
        }
        const unsigned below = (1u << l_) - 1u;
        if (t) tr[bt + pt + __popc(mt & below)] = i;
        if (rr) ro[br + pr + __popc(mr & below)] = i;
        bt += at;
        br += ar;
        __syncthreads();  // (lc_t / lc_r are rewritten by the next round)
      }
      if (tid == 0) {
        S.n_tr = bt;
        S.n_ro = br;
      }
    }
    __syncthreads();
    const double lt0 = S.link_train, hb0 = S.hbm_train, ft0 = S.flops_train;
    const int cnt = S.count, ntr = S.n_tr, nro = S.n_ro;
    const double cur = (T.link > 0 ? div_rn_recip2(lt0, T.link, T.y_link) : 0) +
                       div_rn_recip2(T.hbm - hb0, T.hbm, T.y_hbm);
    Cand best{1e-12, INT_MAX};
    for (int i = crank * nth + tid; i < n; i += nth * csize) {  // single moves (this CTA's share)
      const bool to_train = !in_tr[i];
      if (to_train && cnt + 1 == n) continue;
      if (!to_train && cnt == 1) continue;
      const double ftm = ft0 + (to_train ? uf[i] : -uf[i]);
      if (!in_band(frac(ftm))) continue;
      double lt = lt0;
      if (to_train) lt += ltt[i] + ui[i];
      else lt -= ltt[i] + ui[i];
      const double hbm = hb0 + (to_train ? uh[i] : -uh[i]);
      const double obj = (T.link > 0 ? div_rn_recip2(lt, T.link, T.y_link) : 0) +
                         div_rn_recip2(T.hbm - hbm, T.hbm, T.y_hbm);
      const Cand c{obj - cur, i};
      if (c.gain > best.gain) best = c;  // i ascending per thread: strict '>' keeps the first
    }
    // swaps, scan order a in train ascending, b in rollout ascending: one warp per row a,
    // lanes over b; lb = link_to_train + internal per unit for this step
    double* lb = key;  // free after the ordering
    for (int i = tid; i < n; i += nth) lb[i] = ltt[i] + ui[i];
    __syncthreads();
    const int lane = tid & 31, warp = tid >> 5, nwarps = nth >> 5;
    for (int ia = crank * nwarps + warp; ia < ntr; ia += nwarps * csize) {
      const int a = tr[ia];
      const double Fa = ft0 - uf[a];  // (flops_train - f[a]) + f[b]
      const double Xa = lt0 - lb[a];  // ((link_train - (ltt[a]+int[a])) + (ltt[b]+int[b])) - cross
      const double Ha = hb0 - uh[a];  // (hbm_train - hbm[a]) + hbm[b]
      const double* crow = u.cross + (size_t)a * n;
      for (int ib = lane; ib < nro; ib += 32) {
        const int b = ro[ib];
        if (!in_band(frac(Fa + uf[b]))) continue;
        const double lt = Xa + lb[b] - crow[b];
        const double hbm = Ha + uh[b];
        const double obj = (T.link > 0 ? div_rn_recip2(lt, T.link, T.y_link) : 0) +
                           div_rn_recip2(T.hbm - hbm, T.hbm, T.y_hbm);
        const Cand c{obj - cur, n + a * n + b};
        if (c.gain > best.gain) best = c;
      }
    }
    Cand w = block_best(best, red);
    if (csize > 1) {  // the cluster's best: each warp reads the CTAs' winners (lane k: rank k)
      cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
      if (tid == 0) cbest[par] = w;
      cl.sync();  // (a CTA rewrites cbest[par] two steps later, after the next barrier)
      Cand c{-1e300, INT_MAX};
      if (lane < csize) c = *cl.map_shared_rank(&cbest[par], lane);
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        Cand d;
        d.gain = __shfl_xor_sync(0xffffffffu, c.gain, o);
        d.pos = __shfl_xor_sync(0xffffffffu, c.pos, o);
        if (cand_better(d, c)) c = d;
      }
      w.gain = __shfl_sync(0xffffffffu, c.gain, 0);
      w.pos = __shfl_sync(0xffffffffu, c.pos, 0);
      par ^= 1;
    }
    if (w.pos == INT_MAX) break;
    ++steps;
    if (w.pos < n) {
      if (in_tr[w.pos]) remove(w.pos);
      else add(w.pos);
    } else {
      const int a = (w.pos - n) / n, b = (w.pos - n) % n;
      swap_units(a, b);
    }
  }
  __syncthreads();
  if (csize > 1) cooperative_groups::this_cluster().sync();  // no CTA leaves while its cbest may be read
  if (crank != 0) return;
  for (int i = tid; i < n; i += nth) in_train_out[(size_t)rid * n + i] = ok ? in_tr[i] : 0;
  if (tid == 0) {
    RestartOut o;
    o.ok = ok;
    o.count = S.count;
    o.steps = steps;
    o.obj = (T.link > 0 ? div_rn_recip2(S.link_train, T.link, T.y_link) : 0) +
            div_rn_recip2(T.hbm - S.hbm_train, T.hbm, T.y_hbm);
    out[rid] = o;
  }
}

__global__ void k5_unpack_offers(const Offer* __restrict__ of, const RestartOut* __restrict__ ro, int n_off,
                                 bool exact, double* __restrict__ objs, int* __restrict__ valid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_off) return;
  objs[i] = exact ? of[i].obj : ro[i].obj;
  valid[i] = exact ? of[i].valid : ro[i].ok;
}

// ---------------------------------------------------------------- K5d TopK
struct TopItem {
  double obj;
  int count;     // train devices
  int src;       // offer index
};

struct TopKOut {
  int n_items;
  int pad;
  TopItem item[64];
};

// One warp per offer: its train device ids (sorted: units hold ascending, contiguous
// ids) and its per-machine footprint (TopK's equivalence key, src/partition.cpp:186-190).
__global__ void k5_offer_lists(Units u, const unsigned char* __restrict__ in_train,
                               const int* __restrict__ valid, int n_offers, const int* __restrict__ dmachine,
                               int M, int N, int* __restrict__ ids, int* __restrict__ counts,
                               int* __restrict__ foot) {
  const int o = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (o >= n_offers) return;
  int* f = foot + (size_t)o * M;
  for (int m = lane; m < M; m += 32) f[m] = 0;
  __syncwarp();
  if (!valid[o]) {
    if (lane == 0) counts[o] = 0;
    return;
  }
  int base = 0;
  for (int c = 0; c < u.n; c += 32) {
    const int i = c + lane;
    const bool t = i < u.n && in_train[(size_t)o * u.n + i];
    const int nm = t ? u.mem_off[i + 1] - u.mem_off[i] : 0;
    int incl = nm;  // inclusive prefix sum of member counts
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    const int excl = base + incl - nm;
    for (int k = 0; k < nm; ++k) {
      const int id = u.mem_ids[u.mem_off[i] + k];
      ids[(size_t)o * N + excl + k] = id;
      atomicAdd(&f[dmachine[id]], 1);
    }
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) counts[o] = base;
}

// warp-cooperative lexicographic a < b
__device__ bool warp_lex_less(const int* a, int na, const int* b, int nb) {
  const int lane = threadIdx.x & 31;
  const int m = na < nb ? na : nb;
  for (int c = 0; c < m; c += 32) {
    const int i = c + lane;
    const bool diff = i < m && a[i] != b[i];
    const unsigned bal = __ballot_sync(0xffffffffu, diff);
    if (bal) {
      const int j = c + __ffs(bal) - 1;
      return a[j] < b[j];
    }
  }
  return na < nb;
}

__device__ bool warp_equal(const int* a, const int* b, int n) {
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < n; c += 32) {
    const int i = c + lane;
    if (__any_sync(0xffffffffu, i < n && a[i] != b[i])) return false;
  }
  return true;
}

// Replays TopK::offer (src/partition.cpp:184-201) in offer order with one warp:
// merge into an equivalent entry (|dobj| <= 1e-12 and same footprint) keeping the
// lexicographically smaller train set (no re-sort), else push_back + sort + trim.
__global__ void k5_topk(const double* __restrict__ objs, const int* __restrict__ valid, int n_offers, int k,
                        int M, int N, const int* __restrict__ ids, const int* __restrict__ counts,
                        const int* __restrict__ foot, TopKOut* __restrict__ out) {
  __shared__ TopItem items[65];
  int n_items = 0;
  for (int o = 0; o < n_offers; ++o) {
    if (!valid[o]) continue;
    const double obj = objs[o];
    const int* oid = ids + (size_t)o * N;
    const int nc = counts[o];
    bool merged = false;
    for (int e = 0; e < n_items && !merged; ++e) {
      if (fabs(items[e].obj - obj) > 1e-12) continue;
      if (!warp_equal(foot + (size_t)items[e].src * M, foot + (size_t)o * M, M)) continue;
      if (warp_lex_less(oid, nc, ids + (size_t)items[e].src * N, items[e].count)) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
          items[e].src = o;
          items[e].count = nc;
        }
        __syncwarp();
      }
      merged = true;
    }
    if (merged) continue;
    if ((threadIdx.x & 31) == 0) items[n_items] = TopItem{obj, nc, o};
    __syncwarp();
    ++n_items;
    for (int i = 1; i < n_items; ++i) {  // std::sort: (objective desc, train asc) is a strict total order
      int j = i;
      while (j > 0) {
        const TopItem x = items[j], y = items[j - 1];
        bool before;
        if (x.obj != y.obj) before = x.obj > y.obj;
        else before = warp_lex_less(ids + (size_t)x.src * N, x.count, ids + (size_t)y.src * N, y.count);
        if (!before) break;
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
          items[j] = y;
          items[j - 1] = x;
        }
        __syncwarp();
        --j;
      }
    }
    if (n_items > k) --n_items;
  }
  if ((threadIdx.x & 31) == 0) {
    out->n_items = n_items;
    for (int e = 0; e < n_items; ++e) out->item[e] = items[e];
  }
}

// compute_fraction (src/partition.cpp:361-367) for each result + its train ids
__global__ void k5_emit(const TopKOut* __restrict__ tk, const int* __restrict__ ids, int N,
                        const double* __restrict__ dflops, int* __restrict__ ids_out,
                        double* __restrict__ frac_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double total = 0;
  for (int d = 0; d < N; ++d) total += dflops[d];
  int off = 0;
  for (int e = 0; e < tk->n_items; ++e) {
    const int src = tk->item[e].src, c = tk->item[e].count;
    double t = 0;
    for (int i = 0; i < c; ++i) {
      const int id = ids[(size_t)src * N + i];
      ids_out[off + i] = id;
      t += dflops[id];
    }
    frac_out[e] = t / total;
    off += c;
  }
}

// partition_objective (src/partition.cpp:354-358): State built by add() in the given order
__global__ void k5_objective(const int* __restrict__ train, int nt, const double* __restrict__ dflops,
                             const double* __restrict__ dhbm, const double* __restrict__ links, int N,
                             double* __restrict__ ltt, double* __restrict__ out) {
  __shared__ double s_lt, s_hb;
  if (threadIdx.x == 0) s_lt = s_hb = 0;
  for (int j = threadIdx.x; j < N; j += blockDim.x) ltt[j] = 0;
  __syncthreads();
  for (int k = 0; k < nt; ++k) {
    const int i = train[k];
    if (threadIdx.x == 0) {
      s_lt += ltt[i] + 0.0;  // device units: internal link 0
      s_hb += dhbm[i];
    }
    __syncthreads();
    for (int j = threadIdx.x; j < N; j += blockDim.x)
      if (j != i) ltt[j] += links[(size_t)i * N + j];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double tl = 0, th = 0;
    for (int i = 0; i < N; ++i) {
      tl += 0.0;
      for (int j = i + 1; j < N; ++j) tl += links[(size_t)i * N + j];
    }
    for (int i = 0; i < N; ++i) th += dhbm[i];
    const double lf = tl > 0 ? s_lt / tl : 0;
    out[0] = lf + (th - s_hb) / th;
    double tf = 0, trf = 0;
    for (int d = 0; d < N; ++d) tf += dflops[d];
    for (int k = 0; k < nt; ++k) trf += dflops[train[k]];
    out[1] = trf / tf;
  }
}

// compute_fraction (src/partition.cpp:361-367): two sequential folds
__global__ void k5_fraction(const int* __restrict__ train, int nt, const double* __restrict__ dflops, int N,
                            double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double total = 0, tr = 0;
  for (int d = 0; d < N; ++d) total += dflops[d];
  for (int i = 0; i < nt; ++i) tr += dflops[train[i]];
  *out = tr / total;
}

// ===================================================================== host

template <typename T>
static T* carve3(char*& p, size_t count) {
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
  T* r = reinterpret_cast<T*>(p);
  p += sizeof(T) * count;
  return r;
}

// Unit tables of one granularity (device or machine units): cluster-only data.
struct PartCache {
  int n = 0;
  void* buf = nullptr;
  int* off = nullptr;
  int* ids = nullptr;
  double *uf = nullptr, *uh = nullptr, *ui = nullptr, *base = nullptr, *cross = nullptr;
  Totals* tot = nullptr;
  ~PartCache() {
    if (buf) cudaFree(buf);
  }
};

void part_cache_free(gp_ctx* ctx) {
  for (auto& p : ctx->part_cache) {
    delete static_cast<PartCache*>(p);
    p = nullptr;
  }
}

// graph_partition_candidates (src/partition.cpp:369-406) for q bands in one go (the
// scheduler's iteration-1 probes): unit tables once per context, the restarts of every band
// in ONE k5_restart launch (q x restarts CTAs), the per-band offer / top-k kernels queued
// back to back, one synchronisation and one D2H for all bands. Band i's candidates go to
// out[i * k ..] with their train ids at train_ids[i * k * N ..]; rcs[i] = GP_OK or
// GP_BAND_INFEASIBLE.
// GPLAN_PROFILE=1: partition calls, bands, wall time and k5_restart device time (stderr)
namespace {
struct PartStats {  // (contexts may be driven from several host threads: atomics)
  std::atomic<long long> calls{0}, bands{0};
  AtomicD wall_s, restart_ms;
  ~PartStats() {
    if (std::getenv("GPLAN_PROFILE"))
      std::fprintf(stderr, "partition: %lld calls, %lld bands, %.3f s wall, k5_restart %.3f s\n", calls.load(),
                   bands.load(), (double)wall_s, (double)restart_ms / 1e3);
  }
} g_part_stats;
}  // namespace

int partition_candidates_batch(gp_ctx* ctx, int q, const gp_gamma* gs, const gp_part_opts* o, int k,
                               gp_partition* out, int32_t* train_ids, int32_t* n_out, int* rcs) {
  const int N = ctx->N, M = ctx->M;
  static const bool prof = std::getenv("GPLAN_PROFILE") != nullptr;
  const auto t_call = std::chrono::steady_clock::now();
  cudaEvent_t pe[2] = {nullptr, nullptr};
  for (int i = 0; i < q; ++i) {
    n_out[i] = 0;
    rcs[i] = GP_OK;
  }
  if (q <= 0) return GP_OK;
  if (N < 2) return set_error(GP_INVALID, "graph_partition requires at least two devices");
  if (k < 1 || k > 64) return set_error(GP_INVALID, "k must lie in [1, 64]");
  if (o->restarts < 0) return set_error(GP_INVALID, "restarts must be >= 0");
  // units: machines (device ids ascending) or devices (build_units, src/partition.cpp:37-52)
  const bool by_machine = o->machine_granularity && M >= 2;
  std::vector<int> mem_off, mem_ids;
  if (by_machine) {
    std::vector<std::vector<int>> mm(M);
    for (int d = 0; d < N; ++d) mm[ctx->h_machine[d]].push_back(d);
    for (int m = 0; m < M; ++m) {
      mem_off.push_back((int)mem_ids.size());
      mem_ids.insert(mem_ids.end(), mm[m].begin(), mm[m].end());
    }
  } else {
    for (int d = 0; d < N; ++d) {
      mem_off.push_back(d);
      mem_ids.push_back(d);
    }
  }
  mem_off.push_back((int)mem_ids.size());
  const int n = (int)mem_off.size() - 1;
  if (n > kMaxUnits) return set_error(GP_INVALID, "too many partition units for the sm_100a kernel");
  const bool exact = !o->force_local_search && n <= o->exact_threshold && n <= 20;
  const int n_offers = exact ? (int)((1ull << n) - 2) : o->restarts;
  // ---- unit tables: built once per (context, granularity) — they depend only on the cluster
  PartCache*& pc = reinterpret_cast<PartCache**>(ctx->part_cache)[by_machine ? 1 : 0];
  if (!pc) {
    pc = new PartCache();
    pc->n = n;
    size_t ub = 0;
    auto uadd = [&](size_t b) { ub += ((b + 255) & ~size_t(255)) + 256; };
    uadd(sizeof(int) * (n + 1));
    uadd(sizeof(int) * N);
    uadd(sizeof(double) * n * 4);
    uadd(sizeof(double) * (size_t)n * n);
    uadd(sizeof(Totals));
    GP_CUDA(cudaMalloc(&pc->buf, ub));
    char* qp = static_cast<char*>(pc->buf);
    pc->off = carve3<int>(qp, n + 1);
    pc->ids = carve3<int>(qp, N);
    pc->uf = carve3<double>(qp, n);
    pc->uh = carve3<double>(qp, n);
    pc->ui = carve3<double>(qp, n);
    pc->base = carve3<double>(qp, n);
    pc->cross = carve3<double>(qp, (size_t)n * n);
    pc->tot = carve3<Totals>(qp, 1);
    const size_t in_bytes = (size_t)((char*)(pc->ids + N) - (char*)pc->off);
    char* hp0 = static_cast<char*>(ctx_pinned(ctx, in_bytes + 64));
    if (!hp0) return GP_CUDA_ERROR;
    GP_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(hp0, mem_off.data(), sizeof(int) * (n + 1));
    std::memcpy(hp0 + ((char*)pc->ids - (char*)pc->off), mem_ids.data(), sizeof(int) * N);
    GP_CUDA(cudaMemcpyAsync(pc->off, hp0, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
    ctx->h2d_bytes += (long long)in_bytes;
    const Units u0{n, pc->uf, pc->uh, pc->ui, pc->cross, pc->off, pc->ids};
    k5_units<<<n, 128, 0, ctx->stream>>>(n, pc->off, pc->ids, ctx->d_flops, ctx->d_hbm_bw, ctx->d_links, N,
                                        pc->uf, pc->uh, pc->ui, pc->cross);
    k5_totals<<<1, 256, 0, ctx->stream>>>(u0, pc->tot, pc->base);
    ctx->launches += 2;
    GP_CUDA(cudaGetLastError());
  }
  const Units u{n, pc->uf, pc->uh, pc->ui, pc->cross, pc->off, pc->ids};
  Totals* d_tot = pc->tot;
  double* d_base = pc->base;
  // ---- per-call buffers (q bands)
  const int no1 = std::max(n_offers, 1);
  // per-band result record: TopKOut, train ids, fractions (8-byte aligned), padded to 256 B
  const size_t ids_end = sizeof(TopKOut) + sizeof(int) * (size_t)N * k;
  const size_t frac_off = (ids_end + 7) & ~size_t(7);
  const size_t out_band = (frac_off + sizeof(double) * k + 255) & ~size_t(255);
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += ((b + 255) & ~size_t(255)) + 256; };
  add(sizeof(double2) * q);
  add(sizeof(Offer) * no1);
  add(sizeof(RestartOut) * (size_t)q * std::max(o->restarts, 1));
  add((size_t)q * no1 * n);
  add(sizeof(double) * (size_t)q * no1);
  add(sizeof(int) * (size_t)q * no1);
  add(sizeof(int) * (size_t)q * no1 * N);  // train id lists per offer
  add(sizeof(int) * (size_t)q * no1);      // counts
  add(sizeof(int) * (size_t)q * no1 * M);  // footprints
  add(out_band * q);                        // per band: TopKOut, train ids, fractions
  char* base = static_cast<char*>(ctx_scratch(ctx, bytes, kArenaPartition));
  if (!base) return GP_CUDA_ERROR;
  char* p = base;
  double2* d_bands = carve3<double2>(p, q);
  Offer* d_offer = carve3<Offer>(p, no1);
  RestartOut* d_rout = carve3<RestartOut>(p, (size_t)q * std::max(o->restarts, 1));
  unsigned char* d_mask = carve3<unsigned char>(p, (size_t)q * no1 * n);
  double* d_objs = carve3<double>(p, (size_t)q * no1);
  int* d_valid = carve3<int>(p, (size_t)q * no1);
  int* d_lists = carve3<int>(p, (size_t)q * no1 * N);
  int* d_counts = carve3<int>(p, (size_t)q * no1);
  int* d_foot = carve3<int>(p, (size_t)q * no1 * M);
  char* d_res = carve3<char>(p, out_band * q);
  const size_t mask_bytes = exact ? (size_t)no1 * n : 0;
  const size_t hb_off = (std::max(out_band * q, mask_bytes) + 255) & ~size_t(255);
  char* hp = static_cast<char*>(ctx_pinned(ctx, hb_off + sizeof(double2) * q + 1024));
  if (!hp) return GP_CUDA_ERROR;
  GP_CUDA(cudaStreamSynchronize(ctx->stream));  // (the pinned staging buffer is reused)
  double2* hb = reinterpret_cast<double2*>(hp + hb_off);
  for (int i = 0; i < q; ++i) hb[i] = make_double2(gs[i].gamma_l - o->band_epsilon, gs[i].gamma_h + o->band_epsilon);
  GP_CUDA(cudaMemcpyAsync(d_bands, hb, sizeof(double2) * q, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += (long long)(sizeof(double2) * q);
  if (exact) {
    // masks 1..2^n-2 ascending; the unit membership of mask m is its bit pattern (shared by
    // every band: only the in-band test differs)
    for (int m = 0; m < n_offers; ++m)
      for (int i = 0; i < n; ++i) hp[(size_t)m * n + i] = (char)(((m + 1) >> i) & 1);
    for (int b = 0; b < q; ++b)
      GP_CUDA(cudaMemcpyAsync(d_mask + (size_t)b * no1 * n, hp, mask_bytes, cudaMemcpyHostToDevice, ctx->stream));
    ctx->h2d_bytes += (long long)(mask_bytes * q);
  } else if (o->restarts > 0) {
    const size_t sm = sizeof(double) * 5 * n + sizeof(int) * (3 * n + 2) + n + 64;
    if (sm > 227 * 1024) return set_error(GP_INVALID, "partition units exceed shared memory");
    GP_CUDA(cudaFuncSetAttribute(k5_restart, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    // cluster size: CTAs per restart so that the launch fills the SMs once (one 1024-thread
    // CTA per SM), at most 8 (portable); GPLAN_K5_CLUSTER=c forces c (tests)
    const int n_rs = q * o->restarts;
    int csize = 1;
    while (csize < 8 && (long long)n_rs * csize * 2 <= ctx->num_sms) csize *= 2;
    if (const char* e = std::getenv("GPLAN_K5_CLUSTER")) csize = std::max(1, std::min(8, std::atoi(e)));
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)(n_rs * csize));
    lc.blockDim = dim3(kK5Threads);
    lc.dynamicSmemBytes = sm;
    lc.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    if (prof) {
      cudaEventCreate(&pe[0]);
      cudaEventCreate(&pe[1]);
      cudaEventRecord(pe[0], ctx->stream);
    }
    GP_CUDA(cudaLaunchKernelEx(&lc, k5_restart, u, (const Totals*)d_tot, (const double*)d_base,
                               (const double2*)d_bands, o->restarts, (unsigned long long)o->seed, d_mask, d_rout,
                               csize));
    if (prof) cudaEventRecord(pe[1], ctx->stream);
    ctx->launches++;
  }
  GP_CUDA(cudaGetLastError());
  for (int b = 0; b < q; ++b) {
    const size_t ob = (size_t)b * no1;
    char* rb = d_res + out_band * b;
    TopKOut* d_tk = reinterpret_cast<TopKOut*>(rb);
    int* d_tids = reinterpret_cast<int*>(rb + sizeof(TopKOut));
    double* d_frac = reinterpret_cast<double*>(rb + frac_off);
    if (exact) {
      k5_exact<<<(n_offers + 255) / 256, 256, 0, ctx->stream>>>(u, d_tot, hb[b].x, hb[b].y, d_offer);
      ctx->launches++;
    }
    k5_unpack_offers<<<(n_offers + 255) / 256, 256, 0, ctx->stream>>>(d_offer, d_rout + (size_t)b * o->restarts,
                                                                      n_offers, exact, d_objs + ob, d_valid + ob);
    k5_offer_lists<<<(n_offers + 7) / 8, 256, 0, ctx->stream>>>(u, d_mask + ob * n, d_valid + ob, n_offers,
                                                                ctx->d_machine, M, N, d_lists + ob * N,
                                                                d_counts + ob, d_foot + ob * M);
    k5_topk<<<1, 32, 0, ctx->stream>>>(d_objs + ob, d_valid + ob, n_offers, k, M, N, d_lists + ob * N,
                                       d_counts + ob, d_foot + ob * M, d_tk);
    k5_emit<<<1, 1, 0, ctx->stream>>>(d_tk, d_lists + ob * N, N, ctx->d_flops, d_tids, d_frac);
    ctx->launches += 4;
  }
  GP_CUDA(cudaGetLastError());
  GP_CUDA(cudaMemcpyAsync(hp, d_res, out_band * q, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->d2h_bytes += (long long)(out_band * q);
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (prof) {
    g_part_stats.calls++;
    g_part_stats.bands += q;
    if (pe[0]) {
      float ms = 0;
      cudaEventElapsedTime(&ms, pe[0], pe[1]);
      g_part_stats.restart_ms += ms;
      cudaEventDestroy(pe[0]);
      cudaEventDestroy(pe[1]);
    }
    g_part_stats.wall_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_call).count();
  }
  for (int b = 0; b < q; ++b) {
    const char* rb = hp + out_band * b;
    const TopKOut* htk = reinterpret_cast<const TopKOut*>(rb);
    const int* hids = reinterpret_cast<const int*>(rb + sizeof(TopKOut));
    const double* hfrac = reinterpret_cast<const double*>(rb + frac_off);
    if (htk->n_items == 0) {
      rcs[b] = GP_BAND_INFEASIBLE;
      continue;
    }
    int off = 0;
    for (int e = 0; e < htk->n_items; ++e) {
      gp_partition& po = out[(size_t)b * k + e];
      po.train_offset = off;
      po.train_count = htk->item[e].count;
      po.objective = htk->item[e].obj;
      po.compute_fraction = hfrac[e];
      std::memcpy(train_ids + (size_t)b * k * N + off, hids + off, sizeof(int32_t) * htk->item[e].count);
      off += htk->item[e].count;
    }
    n_out[b] = htk->n_items;
  }
  return GP_OK;
}

int partition_candidates(gp_ctx* ctx, const gp_gamma* g, const gp_part_opts* o, int k, gp_partition* out,
                         int32_t* train_ids, int32_t* n_out) {
  int rc_band = GP_OK;
  const int rc = partition_candidates_batch(ctx, 1, g, o, k, out, train_ids, n_out, &rc_band);
  if (rc) return rc;
  if (rc_band)
    return set_error(GP_BAND_INFEASIBLE, "no bisection satisfies the compute-fraction band [" +
                                             std::to_string(g->gamma_l) + ", " + std::to_string(g->gamma_h) + "]");
  return GP_OK;
}

int compute_fraction(gp_ctx* ctx, const int32_t* train, int nt, double* frac) {
  const int N = ctx->N;
  for (int i = 0; i < nt; ++i)
    if (train[i] < 0 || train[i] >= N) return set_error(GP_INVALID, "unknown device id");
  char* base = static_cast<char*>(ctx_scratch(ctx, sizeof(int) * (nt + 1) + 1024, kArenaMisc));
  if (!base) return GP_CUDA_ERROR;
  char* p = base;
  int* d_t = carve3<int>(p, nt + 1);
  double* d_out = carve3<double>(p, 1);
  char* hp = static_cast<char*>(ctx_pinned(ctx, sizeof(int) * (nt + 1) + 64));
  if (!hp) return GP_CUDA_ERROR;
  std::memcpy(hp, train, sizeof(int) * nt);
  GP_CUDA(cudaMemcpyAsync(d_t, hp, sizeof(int) * (nt + 1), cudaMemcpyHostToDevice, ctx->stream));
  k5_fraction<<<1, 32, 0, ctx->stream>>>(d_t, nt, ctx->d_flops, N, d_out);
  ctx->launches++;
  GP_CUDA(cudaGetLastError());
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  GP_CUDA(cudaMemcpyAsync(hp, d_out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  std::memcpy(frac, hp, sizeof(double));
  return GP_OK;
}

int partition_objective(gp_ctx* ctx, const int32_t* train, int nt, double* obj, double* frac) {
  const int N = ctx->N;
  for (int i = 0; i < nt; ++i)
    if (train[i] < 0 || train[i] >= N) return set_error(GP_INVALID, "unknown device id");
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += ((b + 255) & ~size_t(255)) + 256; };
  add(sizeof(int) * (nt + 1));
  add(sizeof(double) * N);
  add(sizeof(double) * 2);
  char* base = static_cast<char*>(ctx_scratch(ctx, bytes, kArenaPartition));
  if (!base) return GP_CUDA_ERROR;
  char* p = base;
  int* d_t = carve3<int>(p, nt + 1);
  double* d_ltt = carve3<double>(p, N);
  double* d_out = carve3<double>(p, 2);
  char* hp = static_cast<char*>(ctx_pinned(ctx, sizeof(int) * (nt + 1) + 64));
  if (!hp) return GP_CUDA_ERROR;
  std::memcpy(hp, train, sizeof(int) * nt);
  GP_CUDA(cudaMemcpyAsync(d_t, hp, sizeof(int) * (nt + 1), cudaMemcpyHostToDevice, ctx->stream));
  k5_objective<<<1, 256, 0, ctx->stream>>>(d_t, nt, ctx->d_flops, ctx->d_hbm_bw, ctx->d_links, N, d_ltt,
                                           d_out);
  ctx->launches++;
  GP_CUDA(cudaGetLastError());
  double* ho = reinterpret_cast<double*>(hp);
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  GP_CUDA(cudaMemcpyAsync(ho, d_out, sizeof(double) * 2, cudaMemcpyDeviceToHost, ctx->stream));
  GP_CUDA(cudaStreamSynchronize(ctx->stream));
  *obj = ho[0];
  *frac = ho[1];
  return GP_OK;
}

}  // namespace gp
