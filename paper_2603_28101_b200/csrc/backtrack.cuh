// K4 -- backtrack ("identifies the optimal partition index k").
//
// b_m = n;  b_{j-1} = parent[j][b_j] = the LOWEST k in [j-1, b_j - 1] with
//     dp[j-1][k] (+) L[k] * G_j(b_j - k) == dp[j][b_j]
// recomputed from the stored dp rows with the exact arithmetic of the DP kernel
// (Tr<>::comb), so the result is bit-identical to a stored argmin table.
// One warp per problem: 32 splits per step, __ballot_sync + __ffs picks the
// lowest matching k; O(m * n / 32) per problem against the DP's O(n^2 m).
#pragma once
#include "dp_batched.cuh"

namespace hp {

constexpr int kK4Warps = 8;

// The group cost c(k) = L[k] * G_j(cur - k) is non-increasing in k (L sorted, F non-decreasing,
// caps only remove low k), and every candidate satisfies v(k) >= c(k) (dp >= 0), so the lowest
// argmin lies at or after the first k in [lo, cur) with c(k) <= target: a warp-wide 32-ary search.
// group size of items [k, cur): cur - k, or Wp[cur] - Wp[k] with aggregation weights (R5)
__device__ __forceinline__ int gsize(const int32_t* __restrict__ gWp, int cur, int k) {
  return gWp ? gWp[cur] - gWp[k] : cur - k;
}

template <int DT, int SR>
__device__ int first_within_target(const typename Tr<DT, SR>::L* __restrict__ gL,
                                   const typename Tr<DT, SR>::G* __restrict__ grow, int lo, int cur,
                                   typename Tr<DT, SR>::D target, int lane, const int32_t* __restrict__ gWp) {
  using T = Tr<DT, SR>;
  int a0 = lo, b0 = cur;   // first k in [a0, b0) with c(k) <= target; b0 = none
  while (b0 - a0 > 32) {
    const int step = (b0 - a0 + 31) / 32;
    const int k = a0 + lane * step;
    const bool ok = k < b0 && T::norm(T::comb(T::zero(), gL[k], grow[gsize(gWp, cur, k)])) <= target;
    const unsigned msk = __ballot_sync(0xffffffffu, ok);
    if (msk == 0) {   // every probe made failed: continue past the last one actually made
      a0 += min(31, (b0 - 1 - a0) / step) * step + 1;
      continue;
    }
    const int t = __ffs(msk) - 1;
    if (t == 0) { b0 = a0; break; }
    const int na = a0 + (t - 1) * step + 1;
    b0 = a0 + t * step;
    a0 = na;
  }
  if (b0 - a0 > 0) {
    const int k = a0 + lane;
    const bool ok = k < b0 && T::norm(T::comb(T::zero(), gL[k], grow[gsize(gWp, cur, k)])) <= target;
    const unsigned msk = __ballot_sync(0xffffffffu, ok);
    b0 = msk ? a0 + __ffs(msk) - 1 : b0;
  }
  return b0;
}

// lower split bound of layer j's group ending at cur: j-1, the size cap, the kv cap (R6)
template <int DT, bool KV>
__device__ int split_lower_bound(const SolveArgs& a, int b, int j, int cur, const typename SpT<DT>::type* gSp,
                                 const int32_t* gWp) {
  using S = typename SpT<DT>::type;
  int lo = j - 1;
  const int cap = a.caps ? a.caps[(int64_t)b * a.cs + j - 1] : -1;
  if (cap >= 0) {
    if (!gWp) {
      lo = max(lo, cur - cap);
    } else {   // smallest k with Wp[cur] - Wp[k] <= cap (monotone in k)
      int l = lo, h = cur;
      while (l < h) {
        const int mid = (l + h) >> 1;
        if (gWp[cur] - gWp[mid] <= cap) h = mid; else l = mid + 1;
      }
      lo = l;
    }
  }
  if constexpr (KV) {
    const int64_t kvc = a.kv[(int64_t)b * a.kvs + j - 1];
    if (kvc >= 0) {
      int l = lo, h = cur;   // smallest k with Sp[cur] - Sp[k] <= kv (monotone in k)
      while (l < h) {
        const int mid = (l + h) >> 1;
        if (gSp[cur] - gSp[mid] <= (S)kvc) h = mid; else l = mid + 1;
      }
      lo = l;
    }
  }
  return lo;
}

template <int DT, int SR, bool KV, bool W = false>
__global__ void __launch_bounds__(32 * kK4Warps) k4_backtrack(SolveArgs a, int32_t* bounds) {
  using T = Tr<DT, SR>;
  using L = typename T::L;
  using G = typename T::G;
  using D = typename T::D;
  using S = typename SpT<DT>::type;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * kK4Warps + (threadIdx.x >> 5);
  if (b >= a.B) return;
  const int N = a.n, M = a.m, n = prob_n(a, b), m = prob_m(a, b);   // N, M: strides; n, m: this problem's
  int32_t* out = bounds + (int64_t)b * (M + 1);
  if (a.status[b] != HEDDLE_OK) {
    for (int j = lane; j <= M; j += 32) out[j] = -1;
    return;
  }
  for (int j = m + 1 + lane; j <= M; j += 32) out[j] = -1;   // ragged batch: unused tail
  const L* gL = reinterpret_cast<const L*>(a.lengths) + (int64_t)b * a.ls;
  const D* gdp = reinterpret_cast<const D*>(a.dpws) + (int64_t)b * (M + 1) * (N + 1);
  const G* gtab = reinterpret_cast<const G*>(a.gtab);
  const S* gSp = KV ? reinterpret_cast<const S*>(a.spws) + (int64_t)b * (N + 1) : nullptr;
  const int32_t* gWp = W ? a.wpws + (int64_t)b * (N + 1) : nullptr;
  int cur = n;
  if (lane == 0) out[m] = n;
  for (int j = m; j >= 2; --j) {
    const D target = gdp[(int64_t)j * (n + 1) + cur];
    const int d = a.degrees[(int64_t)b * a.ds + j - 1];
    int row = 0;
    for (int q = 0; q < a.D; ++q) row = (a.prof_deg[q] == d) ? q : row;
    const G* grow = gtab + (int64_t)row * a.gstride;
    int lo = split_lower_bound<DT, KV>(a, b, j, cur, gSp, gWp);
    lo = first_within_target<DT, SR>(gL, grow, lo, cur, target, lane, gWp);
    int found = -1;
    for (int base = lo; base < cur && found < 0; base += 32) {
      const int k = base + lane;
      bool hit = false;
      if (k < cur) hit = (T::norm(T::comb(gdp[(int64_t)(j - 1) * (n + 1) + k], gL[k], grow[gsize(gWp, cur, k)])) == target);
      const unsigned msk = __ballot_sync(0xffffffffu, hit);
      if (msk) found = base + __ffs(msk) - 1;
    }
    if (found < 0) {   // unreachable: the target is one of these candidates
      for (int q = lane; q <= M; q += 32) out[q] = -1;
      return;
    }
    cur = found;
    if (lane == 0) out[j - 1] = cur;
  }
  if (lane == 0) out[0] = 0;
}

// One CTA (kK4CtaThreads threads) per problem: for few, large problems (n = 65536), where the
// lowest-argmin scan of min-plus can cover tens of thousands of splits per layer.
constexpr int kK4CtaThreads = 512;
constexpr int kK4PerThread = 8;

template <int DT, int SR, bool KV, bool W = false>
__global__ void __launch_bounds__(kK4CtaThreads) k4_backtrack_cta(SolveArgs a, int32_t* bounds) {
  using T = Tr<DT, SR>;
  using L = typename T::L;
  using G = typename T::G;
  using D = typename T::D;
  using S = typename SpT<DT>::type;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.x;
  const int N = a.n, M = a.m, n = prob_n(a, b), m = prob_m(a, b);
  int32_t* out = bounds + (int64_t)b * (M + 1);
  if (a.status[b] != HEDDLE_OK) {
    for (int j = tid; j <= M; j += kK4CtaThreads) out[j] = -1;
    return;
  }
  for (int j = m + 1 + tid; j <= M; j += kK4CtaThreads) out[j] = -1;
  __shared__ int s_lo, s_found, s_row;
  const L* gL = reinterpret_cast<const L*>(a.lengths) + (int64_t)b * a.ls;
  const D* gdp = reinterpret_cast<const D*>(a.dpws) + (int64_t)b * (M + 1) * (N + 1);
  const G* gtab = reinterpret_cast<const G*>(a.gtab);
  const S* gSp = KV ? reinterpret_cast<const S*>(a.spws) + (int64_t)b * (N + 1) : nullptr;
  const int32_t* gWp = W ? a.wpws + (int64_t)b * (N + 1) : nullptr;
  int cur = n;
  if (tid == 0) out[m] = n;
  for (int j = m; j >= 2; --j) {
    const D target = gdp[(int64_t)j * (n + 1) + cur];
    if (warp == 0) {
      const int d = a.degrees[(int64_t)b * a.ds + j - 1];
      int row = 0;
      for (int q = 0; q < a.D; ++q) row = (a.prof_deg[q] == d) ? q : row;
      const G* grow = gtab + (int64_t)row * a.gstride;
      int lo = split_lower_bound<DT, KV>(a, b, j, cur, gSp, gWp);
      lo = first_within_target<DT, SR>(gL, grow, lo, cur, target, lane, gWp);
      if (lane == 0) { s_lo = lo; s_row = row; s_found = INT_MAX; }
    }
    __syncthreads();
    const G* grow = gtab + (int64_t)s_row * a.gstride;
    const D* prev = gdp + (int64_t)(j - 1) * (n + 1);
    for (int base = s_lo; base < cur; base += kK4CtaThreads * kK4PerThread) {
      int mine = INT_MAX;
#pragma unroll
      for (int i = 0; i < kK4PerThread; ++i) {
        const int k = base + i * kK4CtaThreads + tid;
        if (mine == INT_MAX && k < cur && T::norm(T::comb(prev[k], gL[k], grow[gsize(gWp, cur, k)])) == target)
          mine = k;
      }
      mine = __reduce_min_sync(0xffffffffu, mine);
      if (lane == 0 && mine != INT_MAX) atomicMin(&s_found, mine);
      __syncthreads();
      const int f = s_found;   // every thread reads before any can write it in the next round
      __syncthreads();
      if (f != INT_MAX) break;
    }
    const int found = s_found;
    __syncthreads();
    if (found == INT_MAX) {   // unreachable: the target is one of these candidates
      for (int q = tid; q <= M; q += kK4CtaThreads) out[q] = -1;
      return;
    }
    cur = found;
    if (tid == 0) out[j - 1] = cur;
  }
  if (tid == 0) out[0] = 0;
}


// State query (heddle_place_query): for sampled states (b, j, i) of the last solve, the stored
// dp[j][i] and its back-pointer parent[j][i] = the lowest k in [j-1, i-1] attaining it (R3),
// recomputed from row j-1 exactly as K4 does for the states on the optimal path.  One warp per
// query.  Out-of-region states (i outside [j, n-m+j], R8), failed problems and infeasible states
// give parent -1 and dp = the dtype's infinity (U32 MINPLUS: UINT64_MAX, as the objective).
template <int DT, int SR, bool KV, bool W = false>
__global__ void __launch_bounds__(32 * kK4Warps) k4_query(SolveArgs a, int nq, const int32_t* __restrict__ qb,
                                                         const int32_t* __restrict__ qj,
                                                         const int32_t* __restrict__ qi, void* dp_out,
                                                         int32_t* __restrict__ par_out) {
  using T = Tr<DT, SR>;
  using L = typename T::L;
  using G = typename T::G;
  using D = typename T::D;
  using S = typename SpT<DT>::type;
  const int lane = threadIdx.x & 31;
  const int q = blockIdx.x * kK4Warps + (threadIdx.x >> 5);
  if (q >= nq) return;
  const int N = a.n, M = a.m;
  const int b = qb[q], j = qj[q], cur = qi[q];
  const int m = (b >= 0 && b < a.B) ? prob_m(a, b) : 0;
  const int n = (b >= 0 && b < a.B) ? prob_n(a, b) : 0;
  D val = T::inf();
  int found = -1;
  const bool ok = b >= 0 && b < a.B && j >= 1 && j <= m && cur >= j && cur <= n - m + j &&
                  (j < m || cur == n || m == 1) && a.status[b] == HEDDLE_OK;
  if (ok) {
    const D* gdp = reinterpret_cast<const D*>(a.dpws) + (int64_t)b * (M + 1) * (N + 1);
    val = T::norm(gdp[(int64_t)j * (n + 1) + cur]);
    if (val != T::inf()) {
      if (j == 1) {
        found = 0;   // layer 1: the only split is k = 0
      } else {
        const L* gL = reinterpret_cast<const L*>(a.lengths) + (int64_t)b * a.ls;
        const G* gtab = reinterpret_cast<const G*>(a.gtab);
        const S* gSp = KV ? reinterpret_cast<const S*>(a.spws) + (int64_t)b * (N + 1) : nullptr;
        const int32_t* gWp = W ? a.wpws + (int64_t)b * (N + 1) : nullptr;
        const int d = a.degrees[(int64_t)b * a.ds + j - 1];
        int row = 0;
        for (int r = 0; r < a.D; ++r) row = (a.prof_deg[r] == d) ? r : row;
        const G* grow = gtab + (int64_t)row * a.gstride;
        int lo = split_lower_bound<DT, KV>(a, b, j, cur, gSp, gWp);
        lo = first_within_target<DT, SR>(gL, grow, lo, cur, val, lane, gWp);
        for (int base = lo; base < cur && found < 0; base += 32) {
          const int k = base + lane;
          bool hit = false;
          if (k < cur) hit = (T::norm(T::comb(gdp[(int64_t)(j - 1) * (n + 1) + k], gL[k], grow[gsize(gWp, cur, k)])) == val);
          const unsigned msk = __ballot_sync(0xffffffffu, hit);
          if (msk) found = base + __ffs(msk) - 1;
        }
      }
    }
  }
  if (lane == 0) {
    par_out[q] = found;
    if constexpr (DT == HEDDLE_U32 && SR == HEDDLE_MINPLUS)
      reinterpret_cast<uint64_t*>(dp_out)[q] = (val == T::inf()) ? ~0ull : val;
    else
      reinterpret_cast<D*>(dp_out)[q] = val;
  }
}

}  // namespace hp
