// K8 -- exact "valley" solver for the min-max DP (full dp rows + boundaries).
//
// Eq. 3 with (+) = max:  dp[j][i] = min_{k in [j-1, i-1]} max(dp[j-1][k], c_i(k)),
// c_i(k) = L[k] * G_j(size of items [k, i)) (+inf over a size / token cap, R6).
//   * c_i(k) is non-increasing in k and non-decreasing in i: L is sorted non-increasing,
//     G_j is non-decreasing in the size (F non-decreasing, P:560 -- checked at init, E_RANGE),
//     rounding is monotone, and the caps only forbid large groups.
//   * A split k is dominated for state i by any k' in (k, i-1] with dp[j-1][k'] <= dp[j-1][k]
//     (no larger on both terms).  So the minimum is unchanged when dp[j-1][k] is replaced by the
//     suffix minimum sm_i(k) = min(dp[j-1][k..i-1]), which is non-decreasing in k.
//   * max(sm_i(k), c_i(k)) therefore falls then rises (a valley): with k* = the first k where
//     sm_i(k) >= c_i(k),  dp[j][i] = min(sm_i(k*), c_i(k*-1))  -- values of the same candidates,
//     so bit-identical to the full scan (pinned on the oracle's tables: test P8).
//   * k* is non-decreasing in i (sm_i shrinks and c_i grows with i): a thread sweeping
//     consecutive states gallops from the previous k*.
//   * lowest argmin: every candidate is >= dp[j][i], so it is attained exactly where
//     c_i(k) <= dp[j][i] (a suffix k >= kappa) and dp[j-1][k] <= dp[j][i]: the first such k.
// With one MP degree for all workers every dp row is non-decreasing and sm_i(k) = dp[j-1][k].
// Mixed degrees give rows with descents (about half the layers of the batched sweep), but only
// near the row's start (the slow workers matter only while groups are tiny): with d = the last
// descent of the row, the row is non-decreasing beyond d, so
//   sm_i(k) = dp[j-1][k]                        for k > d,
//           = min(dp[j-1][k..d+1])  (a suffix-minimum array of the short prefix)  for i-1 > d,
// and only states i <= d+1 need a general range minimum: a linear scan while the prefix is short,
// else per 32-element block each element's bitmask of the strict suffix minima of its block
// prefix (min over [k, e] in a block = the element at the first set bit >= k of mask[e]) plus a
// sparse table over the block minima.
// O(n m log n) per problem instead of O(n^2 m) transitions.  Min-max only (a sum of a rising
// and a falling sequence has no valley).
#pragma once
#include <climits>
#include <cstdint>
#include <type_traits>

#include <cooperative_groups.h>

#include "backtrack.cuh"
#include "dp_batched.cuh"

namespace hp {

// K8 CTA sizes: 128 threads (8 CTAs, 32 warps per SM at <= 64 registers) when problems are
// plentiful; 1024 threads when there are fewer problems than SMs (TP sweeps, single instances)
constexpr int kK8Threads = 128;
constexpr int kK8ThreadsWide = 1024;
constexpr int kK8Cluster = 4;        // CTAs per problem in the cluster variant (few problems)
constexpr int kK8ThreadsMid = 512;   // few problems of at most ~512 states per layer: no idle warps
constexpr int kVBlk = 32;        // range-minimum block (one 32-bit mask per element)
constexpr int kScanPrefix = 64;  // default SolveArgs::vscan: descent prefixes shorter than this are
                                 // scanned state by state (no masks / sparse table built)

__host__ __device__ inline int vblocks(int n) { return (n >> 5) + 1; }          // blocks over indices 0..n
__host__ __device__ inline int vlevels(int nb) { int l = 1; while ((2 << (l - 1)) <= nb) ++l; return l; }  // floor(log2 nb)+1

// Range minimum over the computed region of one dp row (the suffix minimum sm_i(k) = rmq(k, i-1)).
template <class T>
struct RowMin {
  using D = typename T::D;
  const D* v;              // the row
  const D* smd;            // [k] = min(v[k..dlast+1]) for k in [row start, dlast+1]
  const uint32_t* mask;    // [nb*32]: bit t of mask[e] <=> element (e & ~31) + t is a strict suffix
                           //   minimum of its block's prefix ending at e   (e <= dlast only)
  const D* bm;             // [nb] block minima (sparse level 0)
  const D* sp;             // [levels-1][nb] sparse levels >= 1 (level l at sp + (l-1)*nb)
  int nb;
  int dlast;               // last descent v[d] > v[d+1] of the region, < row start if none
  __device__ __forceinline__ D operator()(int k, int e) const {
    if (k > dlast) return v[k];          // non-decreasing from k on
    if (e > dlast) return smd[k];        // [k, e] covers d+1, beyond which nothing is smaller
    const int bk = k >> 5, be = e >> 5;
    if (bk == be) return v[k + __ffs(mask[e] >> (k & 31)) - 1];
    D r = T::vmin(v[k + __ffs(mask[(bk << 5) + 31] >> (k & 31)) - 1], v[(be << 5) + __ffs(mask[e]) - 1]);
    if (be - bk > 1) {
      const int a0 = bk + 1, cnt = be - 1 - a0 + 1, l = 31 - __clz(cnt);
      const D* lv = l == 0 ? bm : sp + (int64_t)(l - 1) * nb;
      r = T::vmin(r, T::vmin(lv[a0], lv[be - 1 - (1 << l) + 1]));
    }
    return r;
  }
};

// smd[k] = min(row[k..hi]) for k in [lo, hi], by one warp (suffix scans of 32, right to left)
template <class T>
__device__ __forceinline__ void suffix_min_warp(const typename T::D* row, int lo, int hi, typename T::D* smd,
                                                int lane) {
  using D = typename T::D;
  D carry = T::inf();
  for (int base = hi - 31;; base -= 32) {
    const int idx = base + lane;
    D x = (idx >= lo) ? row[idx] : T::inf();
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const D y = __shfl_down_sync(0xffffffffu, x, off);
      if (lane + off < 32) x = T::vmin(x, y);
    }
    x = T::vmin(x, carry);
    if (idx >= lo) smd[idx] = x;
    carry = __shfl_sync(0xffffffffu, x, 0);
    if (base <= lo) break;
  }
}

// Masks and minimum of one 32-element block: `vals` and `mask` address the block's first
// element; elements outside [lo, hi] (block-relative) read +inf.
template <class T>
__device__ __forceinline__ void block_masks(const typename T::D* vals, int lo, int hi, uint32_t* mask,
                                            typename T::D* bm) {
  using D = typename T::D;
  auto val = [&](int t) -> D { return (t >= lo && t <= hi) ? vals[t] : T::inf(); };
  uint32_t st = 0;
  for (int t = 0; t < kVBlk; ++t) {
    const D x = val(t);
    while (st) {   // pop the staircase entries not strictly below the new element
      const int h = 31 - __clz(st);
      if (val(h) >= x) st &= ~(1u << h); else break;
    }
    st |= 1u << t;
    mask[t] = st;
  }
  *bm = val(__ffs(st) - 1);
}

// The same masks and minimum of one 32-element block by a whole warp, lane t producing mask[t]:
// bit t, and bit h < t iff vals[h] < min(vals[h+1..t]) (h walks down from 31, vals[h] broadcast),
// so the warp issues ~32 uniform steps instead of one lane's serial staircase.
template <class T>
__device__ __forceinline__ void block_masks_warp(const typename T::D* vals, int lo, int hi, uint32_t* mask,
                                                 typename T::D* bm, int lane) {
  using D = typename T::D;
  const D x = (lane >= lo && lane <= hi) ? vals[lane] : T::inf();
  uint32_t st = 0;
  D run = T::inf();
#pragma unroll
  for (int h = 31; h >= 0; --h) {
    const D vh = __shfl_sync(0xffffffffu, x, h);
    if (h <= lane) {
      if (h == lane || vh < run) st |= 1u << h;   // (t itself always: also when +inf)
      run = T::vmin(run, vh);
    }
  }
  mask[lane] = st;
  D mn = x;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mn = T::vmin(mn, __shfl_xor_sync(0xffffffffu, mn, off));
  if (lane == 0) *bm = mn;
}

// The layer's group cost and the valley search, shared by the shared-memory (K8) and the
// global-memory (K8L) kernels.  Pointers address one problem; sizes are item counts, or weight
// sums with aggregation weights (R5).
template <int DT, bool KV, bool W, bool ROWPAD = false>
struct Valley {   // ROWPAD: `grow` is the worker's row staged for every size 0..n, +inf past the cap
  using T = Tr<DT, HEDDLE_MINMAX>;
  using L = typename T::L;
  using G = typename T::G;
  using D = typename T::D;
  using S = typename SpT<DT>::type;
  const L* sL;
  RowMin<T> rm;      // dp[j-1][*] and its range minimum
  const G* grow;     // worker j's cost-table row
  const S* sSp;      // token prefix sums (KV)
  const int* sWp;    // weight prefix sums (W)
  int ghi;           // largest admissible size (the worker's cap, else the table's end)
  int64_t kvc;       // token cap or < 0
  bool scan_prefix;  // short descent prefix: no masks built (states i <= dlast+1 are scanned by the
                     // caller; an argmin inside the prefix is found by walking it)
  // normalised cost of items [k, i) on worker j (+inf when inadmissible)
  __device__ __forceinline__ D cost(int k, int i) const {
    const int s = W ? sWp[i] - sWp[k] : i - k;
    const G g = (ROWPAD || s <= ghi) ? grow[s] : T::gpad();
    D v;   // L * G in the DP kernels' rounding (Tr<>::comb with dp = 0; no max needed: L, G > 0)
    if constexpr (DT == HEDDLE_F32) v = __fmul_rn(sL[k], g);
    else if constexpr (DT == HEDDLE_F64) v = __dmul_rn(sL[k], g);
    else v = T::norm(sL[k] * g);
    if constexpr (KV) {
      if (kvc >= 0 && sSp[i] - sSp[k] > (S)kvc) v = T::inf();
    }
    return v;
  }
  // dp[j][i] over splits [lo, i-1]; `from` >= lo is a split before which the crossing cannot
  // lie (the previous state's k*); returns the value, the lowest argmin (if wanted) and k*.
  // MONO: row j-1 has no descent (dlast < 0), so every range minimum is the row's own value
  // KARY > 2: wide intervals take KARY - 1 independent probes per step (a chain of log_KARY
  // dependent loads instead of log_2: for K8L, whose probes are L2 round trips)
  template <bool ARG, bool MONO = false, int KARY = 2>
  // hint >= lo: a guess of the crossing (K8L: the same state's crossing in the previous layer);
  // the search gallops from it in the direction the first probe shows, then bisects the bracket
  __device__ __forceinline__ D solve(int lo, int i, int from, int& arg, int& kstar, int hint = -1) const {
    const int hi = i - 1;
    auto R = [&](int k, int e) -> D {
      if constexpr (MONO) return rm.v[k];
      else return rm(k, e);
    };
    // the probes' values are kept: the answer min(rm(k*, hi), cost(k*-1, i)) is usually probed
    D rm_t = T::inf(), c_f = T::inf();
    bool have_cf = false;
    auto crossed = [&](int k) {
      const D r = R(k, hi), c = cost(k, i);
      if (r >= c) { rm_t = r; return true; }
      c_f = c;
      return false;
    };
    int f = max(lo, from) - 1;   // last split known not crossed (or lo - 1)
    int t = hi + 1;              // first split known crossed (or hi + 1)
    if (from > lo) {             // gallop from the previous state's crossing (usually 0-2 away)
      int step = 1;
      for (int p = f + 1; p <= hi; p = f + step, step <<= 1) {
        if (crossed(p)) { t = p; break; }
        f = p;
        have_cf = true;
      }
    } else if (hint >= lo && hint <= hi) {
      if (crossed(hint)) {       // the crossing is at or below the hint: gallop down
        t = hint;
        for (int step = 1;; step <<= 1) {
          const int p = t - step;
          if (p <= f) break;
          if (crossed(p)) { t = p; continue; }
          f = p;
          have_cf = true;
          break;
        }
      } else {                   // above the hint: gallop up
        f = hint;
        have_cf = true;
        for (int step = 1;; step <<= 1) {
          const int p = f + step;
          if (p >= t) break;
          if (crossed(p)) { t = p; break; }
          f = p;
        }
      }
    }                            // else: plain bisection of [lo, hi]
    bool have_rt = t <= hi;
    if constexpr (KARY > 2) {
      while (t - f > 2 * KARY) {
        const int q = (t - f) / KARY;
        D r[KARY - 1], c[KARY - 1];
#pragma unroll
        for (int u = 0; u < KARY - 1; ++u) {
          r[u] = R(f + (u + 1) * q, hi);
          c[u] = cost(f + (u + 1) * q, i);
        }
        int nf = f, nt = t;
#pragma unroll
        for (int u = KARY - 2; u >= 0; --u)   // the lowest crossed probe
          if (r[u] >= c[u]) { nt = f + (u + 1) * q; rm_t = r[u]; have_rt = true; }
#pragma unroll
        for (int u = 0; u < KARY - 1; ++u)    // the highest probe not crossed
          if (!(r[u] >= c[u])) { nf = f + (u + 1) * q; c_f = c[u]; have_cf = true; }
        f = nf;
        t = nt;
      }
    }
    while (t - f > 1) {
      const int mid = (f + t) >> 1;
      if (crossed(mid)) { t = mid; have_rt = true; } else { f = mid; have_cf = true; }
    }
    kstar = t;
    // rm_t / c_f hold the last crossed / not-crossed probe, which are t and f when probed
    D v = (t <= hi) ? (have_rt ? rm_t : R(t, hi)) : T::inf();
    if (t > lo) v = T::vmin(v, have_cf && f == t - 1 ? c_f : cost(t - 1, i));
    if constexpr (ARG) {
      if (v == T::inf()) {
        arg = -1;
      } else {   // attained where cost(k) <= v (k >= kappa) and dp[j-1][k] <= v: the first such k
        int a0 = lo - 1, b0 = hi;              // cost(hi) <= v: the smallest cost
        while (b0 - a0 > 1) {
          const int mid = (a0 + b0) >> 1;
          if (cost(mid, i) <= v) b0 = mid; else a0 = mid;
        }
        const int kappa = b0;
        if (scan_prefix && kappa <= rm.dlast) {   // no masks: walk the short descent prefix
          int e = kappa;                          // (the row is non-decreasing from dlast+1 on, so
          while (rm.v[e] > v) ++e;                //  the first e with v[e] <= v is at most dlast+1)
          arg = e;
        } else {
          a0 = kappa - 1;
          b0 = hi;                                // rm(kappa, hi) <= v
          while (b0 - a0 > 1) {
            const int mid = (a0 + b0) >> 1;
            if (R(kappa, mid) <= v) b0 = mid; else a0 = mid;
          }
          arg = b0;
        }
      }
    }
    return v;
  }
};

// Shared-memory carve-up of the one-CTA-per-problem valley kernel (bytes).
template <int DT>
struct K8Smem {
  using T = Tr<DT, HEDDLE_MINMAX>;
  int lOff, gOff, d0Off, d1Off, smdOff, maskOff, spOff, sspOff, wpOff, rowOff, capOff, kvOff, total;
  __host__ __device__ K8Smem(int n, int m, bool kv, bool w) {
    int o = 0;
    auto take = [&](int bytes) { int at = o; o += (bytes + 15) & ~15; return at; };
    const int nb = vblocks(n);
    lOff = take((int)sizeof(typename T::L) * align4(n + kLPad));
    gOff = w ? -1 : take((int)sizeof(typename T::G) * (n + 1));   // worker's cost row, cap-masked
    d0Off = take((int)sizeof(typename T::D) * nb * kVBlk);
    d1Off = take((int)sizeof(typename T::D) * nb * kVBlk);
    smdOff = take((int)sizeof(typename T::D) * (n + 1));
    maskOff = take(4 * nb * kVBlk);
    spOff = take((int)sizeof(typename T::D) * nb * vlevels(nb));
    sspOff = kv ? take(8 * (n + 1)) : -1;
    wpOff = w ? take(4 * align4(n + kLPad)) : -1;
    rowOff = take(4 * m);
    capOff = take(4 * m);
    kvOff = take(8 * m);
    total = o;
  }
};

// ---------------------------------------------------------------------------- K8: one CTA per problem
// CL > 1: a thread-block cluster of CL CTAs per problem (few problems: the paper's per-call
// shapes).  Every CTA holds the whole problem and the full dp rows; CTA r computes the r-th part
// of each layer's states and stores them into its own row and, over distributed shared memory,
// into the other CTAs' rows; one cluster barrier per layer replaces the CTA barrier.  The range
// minimum of the previous row is rebuilt by every CTA on its own copy; CTA 0 writes the rows to
// the workspace and walks the fused backtrack.
template <int DT, bool KP, bool KV, bool W, int NT, int CL = 1>
__global__ void __launch_bounds__(NT, CL > 1 ? 1 : 1024 / NT) k8_valley(SolveArgs a) {
  using T = Tr<DT, HEDDLE_MINMAX>;
  using L = typename T::L;
  using G = typename T::G;
  using D = typename T::D;
  using S = typename SpT<DT>::type;
  extern __shared__ __align__(16) unsigned char smem[];
  const int N = a.n, M = a.m, b = blockIdx.x / CL, tid = threadIdx.x;   // N, M: strides; n, m: this problem's
  const int cr = CL > 1 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
  const int n = prob_n(a, b), m = prob_m(a, b);
  const K8Smem<DT> lay(N, M, KV, W);
  L* sL = reinterpret_cast<L*>(smem + lay.lOff);
  G* sG = W ? nullptr : reinterpret_cast<G*>(smem + lay.gOff);
  D* const sdp0 = reinterpret_cast<D*>(smem + lay.d0Off);
  D* const sdp1 = reinterpret_cast<D*>(smem + lay.d1Off);
  D* ssmd = reinterpret_cast<D*>(smem + lay.smdOff);
  uint32_t* smask = reinterpret_cast<uint32_t*>(smem + lay.maskOff);
  D* ssp = reinterpret_cast<D*>(smem + lay.spOff);
  S* sSp = KV ? reinterpret_cast<S*>(smem + lay.sspOff) : nullptr;
  int* sWp = W ? reinterpret_cast<int*>(smem + lay.wpOff) : nullptr;
  int* srow = reinterpret_cast<int*>(smem + lay.rowOff);
  int* scap = reinterpret_cast<int*>(smem + lay.capOff);
  int64_t* skv = reinterpret_cast<int64_t*>(smem + lay.kvOff);
  // fused backtrack (a.fbounds): every dp row of the problem, [m+1][n+1], after the carve-up
  D* stab = (a.fbounds && !KP) ? reinterpret_cast<D*>(smem + lay.total) : nullptr;
  __shared__ int s_err, s_dlast[2];
  if (tid == 0) { s_dlast[0] = -1; s_dlast[1] = -1; }
  if (load_problem<DT, HEDDLE_MINMAX, KV, W, NT>(a, b, n, m, sL, srow, scap, skv, sSp, sWp, s_err) != 0) return;
  __syncthreads();
  D* gdp = reinterpret_cast<D*>(a.dpws) + (int64_t)b * (M + 1) * (N + 1);
  int32_t* gpar = KP ? a.parws + (int64_t)b * (M + 1) * (N + 1) : nullptr;
  const G* gtab = reinterpret_cast<const G*>(a.gtab);
  const int nb = vblocks(n);

  for (int j = 1; j <= m; ++j) {
    D* const prev = (j & 1) ? sdp0 : sdp1;
    D* const cur = (j & 1) ? sdp1 : sdp0;
    D* rcur[CL];   // this layer's row in every CTA of the cluster (rcur[cr] = cur)
#pragma unroll
    for (int r = 0; r < CL; ++r) {
      if constexpr (CL > 1) rcur[r] = cooperative_groups::this_cluster().map_shared_rank(cur, r);
      else rcur[r] = cur;
    }
    auto put = [&](int i, D v) {   // a computed state into every copy of the row
      cur[i] = v;
      if constexpr (CL > 1) {
#pragma unroll
        for (int r = 0; r < CL; ++r)
          if (r != cr) rcur[r][i] = v;
      }
    };
    const int ilo = (j == 1) ? 1 : (j == m ? n : j);
    const int ihi = (j == 1 || j < m) ? n - m + j : n;   // m == 1: layer 1 is the last (i up to n)
    int dl = -1;            // last descent of row j-1 (-1: non-decreasing)
    bool scan_prefix = false;
    // worker j's cost row, masked by its cap (restaged only when the profile row or cap changes;
    // the previous layer's reads ended at its last barrier)
    const bool restage = !W && (j == 1 || srow[j - 1] != srow[j - 2] || scap[j - 1] != scap[j - 2]);
    if (restage) {
      const G* grow = gtab + (int64_t)srow[j - 1] * a.gstride;
      const int cap = scap[j - 1], hi = (cap >= 0 && cap < n) ? cap : n;
      for (int t = tid; t <= n; t += NT) sG[t] = (t >= 1 && t <= hi) ? grow[t] : T::gpad();
    }
    if (j == 1 && restage) __syncthreads();
    if (j > 1) {
      // range minimum of row j-1 over its computed region [j-1, n-m+j-1]
      const int plo = j - 1, phi = n - m + j - 1;
      int myd = -1;
      for (int t = plo + tid; t < phi; t += NT)
        if (prev[t] > prev[t + 1]) myd = t;
      myd = __reduce_max_sync(0xffffffffu, myd);
      if ((tid & 31) == 0 && myd >= 0) atomicMax(&s_dlast[j & 1], myd);
      __syncthreads();
      dl = s_dlast[j & 1];
      if (tid == 0) s_dlast[(j + 1) & 1] = -1;          // for layer j+1 (read after its barrier)
      if (dl >= 0) {
        scan_prefix = dl - plo < a.vscan;
        if (tid < 32) suffix_min_warp<T>(prev, plo, dl + 1, ssmd, tid);
        if (!scan_prefix) {   // long descent prefix: masks + sparse table over its blocks
          const int blo = plo >> 5, bhi = dl >> 5;
          for (int blk = blo + (tid - 32); tid >= 32 && blk <= bhi; blk += NT - 32)
            block_masks<T>(prev + (blk << 5), plo - (blk << 5), dl - (blk << 5), smask + (blk << 5), ssp + blk);
          __syncthreads();
          for (int l = 1; (1 << l) <= bhi - blo + 1; ++l) {   // sparse levels over the block minima
            const D* src = ssp + (int64_t)(l - 1) * nb;
            D* dst = ssp + (int64_t)l * nb;
            for (int blk = blo + tid; blk + (1 << l) - 1 <= bhi; blk += NT)
              dst[blk] = T::vmin(src[blk], src[blk + (1 << (l - 1))]);
            __syncthreads();
          }
        }
        __syncthreads();
      }
    }
    const int cap = scap[j - 1];
    Valley<DT, KV, W, !W> V{sL, RowMin<T>{prev, ssmd, smask, ssp, ssp + nb, nb, dl},
                        W ? gtab + (int64_t)srow[j - 1] * a.gstride : sG, sSp, sWp,
                        W ? ((cap >= 0 && cap < a.gstride - 1) ? cap : a.gstride - 1) : n, KV ? skv[j - 1] : -1,
                        scan_prefix};
    if (j == 1) {   // dp[1][i] = L(tau_1) * T * F(i)
      for (int i = ilo + tid; i <= ihi; i += NT) {
        const D v = V.cost(0, i);
        cur[i] = v;
        if (KP) gpar[(int64_t)(n + 1) + i] = (v == T::inf()) ? -1 : 0;
      }
    } else {
      // states before the end of a short descent prefix (i - 1 <= dl): Eq. 3 as written, each by
      // one warp (lanes over the splits, lowest-index argmin), dealt round-robin over the warps
      const int pre_hi = scan_prefix ? min(dl + 1, ihi) : ilo - 1;
      const int lane = tid & 31;
      for (int i = ilo + cr * (NT / 32) + (tid >> 5); i <= pre_hi; i += CL * (NT / 32)) {
        D best = T::inf();
        int bk = INT_MAX;
        for (int k = j - 1 + lane; k < i; k += 32) {
          const D cv = V.cost(k, i), pv = prev[k];
          const D c = pv > cv ? pv : cv;
          if (c < best) { best = c; bk = k; }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const D ov = shfl_down(best, off);
          const int ok = __shfl_down_sync(0xffffffffu, bk, off);
          if (ov < best || (ov == best && ok < bk)) { best = ov; bk = ok; }
        }
        if (lane == 0) {
          put(i, best);
          if (KP) gpar[(int64_t)j * (n + 1) + i] = (best == T::inf()) ? -1 : bk;
        }
      }
      // the other states: contiguous runs per thread, so each search gallops from the previous k*
      // (with a cluster: the CTA's contiguous part of them)
      const int pc = (ihi - pre_hi + CL - 1) / CL;
      const int s0 = pre_hi + 1 + cr * pc;
      const int ns = min(ihi, s0 + pc - 1) - s0 + 1;
      const int per = (max(ns, 0) + NT - 1) / NT;
      const int r0 = s0 + tid * per, r1 = min(s0 + ns - 1, r0 + per - 1);
      int from = j - 1;
      auto run = [&](auto mono) {
        for (int i = r0; i <= r1; ++i) {
          int arg = -1, ks;
          const D v = V.template solve<KP, decltype(mono)::value>(j - 1, i, from, arg, ks);
          from = ks;
          put(i, v);
          if (KP) gpar[(int64_t)j * (n + 1) + i] = arg;
        }
      };
      if (dl < 0) run(std::true_type{}); else run(std::false_type{});   // (uniform per layer)
    }
    if constexpr (CL > 1) cooperative_groups::this_cluster().sync();   // every copy of row j complete
    else __syncthreads();
    // the finished row to the workspace (coalesced) for the backtrack; -1 parents off the region
    if (cr == 0) {
      for (int i = tid; i <= n; i += NT) {
        const bool in = (i >= ilo && i <= ihi);
        if (in) gdp[(int64_t)j * (n + 1) + i] = cur[i];
        if (KP && !in) gpar[(int64_t)j * (n + 1) + i] = -1;
        if (stab && in) stab[(int64_t)j * (n + 1) + i] = cur[i];
      }
    }
    // (cur is read as `prev` by layer j+1 and rewritten by layer j+2, after its barriers; the
    //  masks / sparse levels of row j are built by layer j+1 after this layer's last barrier)
  }
  if (cr != 0) return;   // (the last cluster barrier ended every remote access to this CTA)
  const D obj = ((m & 1) ? sdp1 : sdp0)[n];
  if (tid == 0) {
    const int st = (obj == T::inf()) ? (int)HEDDLE_E_INFEASIBLE : (int)HEDDLE_OK;
    a.status[b] = st;
    if (a.status_out) a.status_out[b] = st;
    reinterpret_cast<D*>(a.objective)[b] = obj;
  }
  if (stab) {   // fused backtrack from the shared-memory table: K4's rule, the lowest k in
                // [lower bound, cur) whose candidate reproduces dp[j][cur] (R3)
    int32_t* out = a.fbounds + (int64_t)b * (M + 1);
    for (int q = m + 1 + tid; q <= M; q += NT) out[q] = -1;
    if (obj == T::inf()) {
      for (int q = tid; q <= m; q += NT) out[q] = -1;
      return;
    }
    __syncthreads();   // the last row of the table (its store loop above) is complete
    __shared__ int s_found;
    // the cost rows come from sG, restaged unmasked when the profile row changes (degrees only grow
    // walking back): the lower bound already excludes the groups over a cap.  Without caps the
    // forward pass left worker m's row unmasked in sG.
    int cur_i = n, staged = (W || a.caps) ? -1 : srow[m - 1];
    if (tid == 0) out[m] = n;
    for (int j = m; j >= 2; --j) {
      if (!W && srow[j - 1] != staged) {
        staged = srow[j - 1];
        __syncthreads();
        const G* grow = gtab + (int64_t)staged * a.gstride;
        for (int t = tid; t <= n; t += NT) sG[t] = t >= 1 ? grow[t] : T::gpad();
      }
      const D target = stab[(int64_t)j * (n + 1) + cur_i];
      const int lo = split_lower_bound<DT, KV>(a, b, j, cur_i, sSp, sWp);
      const G* grow = W ? gtab + (int64_t)srow[j - 1] * a.gstride : sG;
      if (tid == 0) s_found = INT_MAX;
      __syncthreads();
      int mine = INT_MAX;
      for (int k = lo + tid; k < cur_i && mine == INT_MAX; k += NT)
        if (T::norm(T::comb(stab[(int64_t)(j - 1) * (n + 1) + k], sL[k], grow[gsize(sWp, cur_i, k)])) == target)
          mine = k;
      mine = __reduce_min_sync(0xffffffffu, mine);
      if ((tid & 31) == 0 && mine != INT_MAX) atomicMin(&s_found, mine);
      __syncthreads();
      cur_i = s_found;
      __syncthreads();          // every thread has read s_found before thread 0 resets it
      if (cur_i == INT_MAX) {   // unreachable: the target is one of these candidates
        for (int q = tid; q <= m; q += NT) out[q] = -1;
        return;
      }
      if (tid == 0) out[j - 1] = cur_i;
    }
    if (tid == 0) out[0] = 0;
  }
}

// ------------------------------------------------------------ K8L: one launch per layer (large n)
// dp rows live in the workspace (L2-resident per layer).  A warp owns 4 consecutive 32-element
// blocks of the row (a lane: 4 consecutive states, galloping), then builds their masks and minima
// for the next layer.  Validation and prefix sums come from the layered prologue.
#ifndef HEDDLE_K8L_RUN
#define HEDDLE_K8L_RUN 1
#endif
#ifndef HEDDLE_K8L_WARPS
#define HEDDLE_K8L_WARPS 8
#endif
constexpr int kK8LRun = HEDDLE_K8L_RUN;      // consecutive states per lane (= 32-element blocks per warp)
constexpr int kK8LWarps = HEDDLE_K8L_WARPS;
#ifndef HEDDLE_K8L_KARY
#define HEDDLE_K8L_KARY 4
#endif
constexpr int kK8LKary = HEDDLE_K8L_KARY;    // probes + 1 per step of a state's first crossing search

struct ValleyWs {                // K8L range-minimum workspace (per problem, row parity p = j & 1)
  uint32_t* mask;                // [2][B][nb*32]
  void* bm;                      // [2][B][nb]        block minima (sparse level 0)
  void* sp;                      // [B][levels-1][nb] sparse levels >= 1 (rebuilt per row)
  void* smd;                     // [B][max_n+1]      suffix minima of the descent prefix (per row)
  int* dlast;                    // [B]               last descent of the row (-1: none)
  int* dlrun;                    // [2][B]            descents inside the warps' runs (-1; by parity)
  unsigned* done;                // [B]               CTAs of the current layer finished
  int* khint;                    // [2][B][max_n+1]   each state's crossing in the last two layers
  int nbmax, lvmax, nmax;
};

// Row j's range-minimum extras, by the last CTA of layer j to finish (`nt` threads): the last
// descent of the row (the largest of the in-run descents the warps found and the pairs across
// 32-element blocks), the suffix minima of the descent prefix, and sparse levels >= 1 over the
// prefix's block minima.  Reads of row j and of the block minima written by other CTAs of this
// launch go through L2 (ld.cg).
template <class T>
__device__ __forceinline__ void k8l_row_extras(const SolveArgs& a, int j, const ValleyWs& w, int b, int tid, int nt,
                                               int* s_dl) {
  using D = typename T::D;
  const int n = a.n, m = a.m;
  const int ilo = (j == 1) ? 1 : j, ihi = n - m + j, nb = vblocks(n);
  const D* row = reinterpret_cast<const D*>(a.dpws) + ((int64_t)b * (m + 1) + j) * (n + 1);
  int* run_slot = w.dlrun + (int64_t)(j & 1) * a.B + b;
  int myd = -1;
  constexpr int U = 8;   // block-boundary pairs (t = 32 q + 31, t + 1), U pairs of loads in flight
  for (int q0 = (ilo >> 5) + tid; (q0 << 5) + 31 < ihi; q0 += U * nt) {
    D x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = min(((q0 + u * nt) << 5) + 31, ihi - 1);
      x[u] = ld_cg(row + t);
      y[u] = ld_cg(row + t + 1);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = ((q0 + u * nt) << 5) + 31;
      if (t >= ilo && t < ihi && x[u] > y[u]) myd = max(myd, t);
    }
  }
  myd = __reduce_max_sync(0xffffffffu, myd);
  if ((tid & 31) == 0 && myd >= 0) atomicMax(s_dl, myd);
  __syncthreads();
  const int dl = max(*s_dl, ld_cg(run_slot));
  __syncthreads();
  if (tid == 0) {
    w.dlast[b] = dl;
    *run_slot = -1;   // the slot of parity j & 1 is next written by layer j + 2
    w.done[b] = 0;
  }
  if (dl < 0) return;
  if (tid < 32) {   // smd[k] = min(row[k..dl+1]) (suffix scans of 32, right to left)
    D* smd = reinterpret_cast<D*>(w.smd) + (int64_t)b * (n + 1);
    D carry = T::inf();
    for (int base = dl + 1 - 31;; base -= 32) {
      const int idx = base + tid;
      D x = (idx >= ilo) ? ld_cg(row + idx) : T::inf();
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const D y = __shfl_down_sync(0xffffffffu, x, off);
        if (tid + off < 32) x = T::vmin(x, y);
      }
      x = T::vmin(x, carry);
      if (idx >= ilo) smd[idx] = x;
      carry = __shfl_sync(0xffffffffu, x, 0);
      if (base <= ilo) break;
    }
  }
  const int blo = ilo >> 5, bhi = dl >> 5;
  const D* bmj = reinterpret_cast<const D*>(w.bm) + ((int64_t)(j & 1) * a.B + b) * nb;
  D* sp = reinterpret_cast<D*>(w.sp) + (int64_t)b * (w.lvmax - 1) * nb;
  for (int l = 1; (1 << l) <= bhi - blo + 1; ++l) {
    const D* src = l == 1 ? bmj : sp + (int64_t)(l - 2) * nb;
    D* dst = sp + (int64_t)(l - 1) * nb;
    for (int blk = blo + tid; blk + (1 << l) - 1 <= bhi; blk += nt)
      dst[blk] = T::vmin(ld_cg(src + blk), ld_cg(src + blk + (1 << (l - 1))));
    __syncthreads();
  }
}

template <int DT, bool KP, bool KV, bool W = false>
__global__ void __launch_bounds__(32 * kK8LWarps, DT == HEDDLE_F64 ? 2 : 4) k8l_layer(SolveArgs a, int j, ValleyWs w) {
  using T = Tr<DT, HEDDLE_MINMAX>;
  using L = typename T::L;
  using G = typename T::G;
  using D = typename T::D;
  using S = typename SpT<DT>::type;
  __shared__ D s_row[kK8LWarps][32 * kK8LRun];
  __shared__ int s_dl, s_last;
  const int n = a.n, m = a.m, b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // launched with programmatic stream serialisation: wait until the previous layer's grid has
  // completed and its stores are visible (the next layer's grid is released after the states)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int ilo = (j == 1) ? 1 : (j == m ? n : j);
  const int ihi = (j == 1 || j < m) ? n - m + j : n;
  const int blk0 = (ilo >> 5) + kK8LRun * (blockIdx.x * kK8LWarps + warp);
  const bool active = (blk0 << 5) <= ihi;
  const int x0 = (blk0 << 5) + kK8LRun * lane;
  // the per-launch loads issued together (one round trip, not one after another)
  const int status = a.status[b];
  const int2 rc = a.rowcap[(int64_t)b * m + j - 1];   // {profile row, cap} from the prologue
  const int dlast = j > 1 ? w.dlast[b] : -1;
  const int64_t par = (int64_t)a.B * (w.nmax + 1);   // parity stride of the crossing hints
  const int hint0 = (j > 1 && active && x0 <= n) ? w.khint[((j - 1) & 1) * par + (int64_t)b * (w.nmax + 1) + x0] : -1;
  if (status != HEDDLE_OK) return;   // (uniform over the problem's CTAs)
  if (tid == 0) s_dl = -1;
  const int nb = vblocks(n);
  D* gdp = reinterpret_cast<D*>(a.dpws) + (int64_t)b * (m + 1) * (n + 1);
  if (active) {
    const int row = rc.x, cap = rc.y;
    const int pp = (j - 1) & 1;
    const RowMin<T> rm{gdp + (int64_t)(j - 1) * (n + 1), reinterpret_cast<const D*>(w.smd) + (int64_t)b * (n + 1),
                       w.mask + ((int64_t)pp * a.B + b) * nb * kVBlk,
                       reinterpret_cast<const D*>(w.bm) + ((int64_t)pp * a.B + b) * nb,
                       reinterpret_cast<const D*>(w.sp) + (int64_t)b * (w.lvmax - 1) * nb, nb, dlast};
    Valley<DT, KV, W> V{reinterpret_cast<const L*>(a.lengths) + (int64_t)b * a.ls, rm,
                        reinterpret_cast<const G*>(a.gtab) + (int64_t)row * a.gstride,
                        KV ? reinterpret_cast<const S*>(a.spws) + (int64_t)b * (n + 1) : nullptr,
                        W ? a.wpws + (int64_t)b * (n + 1) : nullptr,
                            (cap >= 0 && cap < a.gstride - 1) ? cap : a.gstride - 1,
                            KV ? a.kv[(int64_t)b * a.kvs + j - 1] : -1, false};
    int from = j - 1;
#pragma unroll
    for (int r = 0; r < kK8LRun; ++r) {
      const int i = x0 + r;
      D v = T::inf();
      if (i >= ilo && i <= ihi) {
        int arg = -1, ks = from;
        int* kh = w.khint + (int64_t)b * (w.nmax + 1) + i;
        if (j == 1) {
          v = V.cost(0, i);
          arg = (v == T::inf()) ? -1 : 0;
          kh[par] = -1;   // (layer 1 has no crossing: layer 2 bisects)
        } else {
          // the same state's crossing one layer up: usually a few splits away (K8L is bound by the
          // chain of L2 round trips of this search, not by its instructions)
          const int hint = (r == 0) ? hint0 : -1;
          v = rm.dlast < 0 ? V.template solve<KP, true, kK8LKary>(j - 1, i, from, arg, ks, hint)   // monotone row j-1
                           : V.template solve<KP, false, kK8LKary>(j - 1, i, from, arg, ks, hint);
          from = ks;
          kh[(j & 1) * par] = ks;
        }
        gdp[(int64_t)j * (n + 1) + i] = v;
        if (KP) a.parws[((int64_t)b * (m + 1) + j) * (n + 1) + i] = arg;
      }
      s_row[warp][kK8LRun * lane + r] = v;
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (j == m) return;   // the last row is never queried
  __syncwarp();
  int myd = -1;
  if (active) {
    // masks + minimum of the warp's blocks of row j
    const int p = j & 1;
    uint32_t* mk = w.mask + ((int64_t)p * a.B + b) * nb * kVBlk;
    D* bmj = reinterpret_cast<D*>(w.bm) + ((int64_t)p * a.B + b) * nb;
#pragma unroll
    for (int r = 0; r < kK8LRun; ++r) {
      const int blk = blk0 + r;
      if (blk <= (ihi >> 5))
        block_masks_warp<T>(s_row[warp] + 32 * r, ilo - (blk << 5), ihi - (blk << 5), mk + (blk << 5), bmj + blk, lane);
    }
    // descents v[t] > v[t+1] inside the warp's run (pairs across warps: the last CTA)
#pragma unroll
    for (int r = 0; r < kK8LRun; ++r) {
      const int q = kK8LRun * lane + r, t = x0 + r;
      if (q + 1 < 32 * kK8LRun && t >= ilo && t + 1 <= ihi && s_row[warp][q] > s_row[warp][q + 1]) myd = t;
    }
  }
  myd = __reduce_max_sync(0xffffffffu, myd);
  __syncthreads();   // (s_dl initialised)
  if (lane == 0 && myd >= 0) atomicMax(&s_dl, myd);
  __syncthreads();   // every thread's row / mask / minimum stores precede thread 0's fence
  if (tid == 0) {
    if (s_dl >= 0) atomicMax(w.dlrun + (int64_t)(j & 1) * a.B + b, s_dl);
    // release (the CTA's stores, ordered by the barrier) + acquire (the other CTAs' stores)
    s_last = atom_add_acq_rel_gpu(w.done + b, 1u) == gridDim.x - 1;
    s_dl = -1;
  }
  __syncthreads();
  if (!s_last) return;
  k8l_row_extras<T>(a, j, w, b, tid, 32 * kK8LWarps, &s_dl);
}

}  // namespace hp
