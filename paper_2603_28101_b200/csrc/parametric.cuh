// K7 -- objective-only exact solver for the min-max DP (the parametric
// characterisation pinned as P6 in DESIGN.md §5).
//
// For min-max (Eq. 3) the optimum OPT is the smallest X such that the n sorted
// trajectories can be cut into exactly m non-empty contiguous groups, group j on worker j,
// each costing <= X.  feasible(X) tracks R_j = the prefix ends coverable by exactly j such
// groups; with unit weights R_j is an interval [lo_j, hi_j]:
//   * the cost c_j(a, e) = L[a] * G_j(e - a) of items [a, e) is non-increasing in the start a
//     (L sorted, F non-decreasing, caps / kv caps only forbid large groups), so the cheapest
//     start for an end e is a = min(hi_{j-1}, e - 1);
//   * for e <= hi_{j-1}+1 that is the single item e-1, whose cost is non-increasing in e
//     -> lo_j = first such e with c <= X (and e = hi_{j-1}+1 must qualify, else R_j is empty);
//   * for e >= hi_{j-1}+1 the start is hi_{j-1} and c is non-decreasing in e
//     -> hi_j = last such e with c <= X.
// OPT is found by bisection over the ordered bit patterns of the value type (costs and X are
// compared in the kernel's own arithmetic, Tr<>::comb), so it equals the DP's dp[m][n] bit for
// bit.  One warp per problem; every monotone search is 32-ary (ballot per probe round).
// O(bits * m * log32 n) cost evaluations instead of O(n^2 m) transitions: no partition is
// produced (the canonical lowest-index boundaries still come from the DP), which is exactly
// what the resource manager's makespan evaluations need (Alg. 2).
#pragma once
#include <climits>
#include <cstdint>

#include "dp_batched.cuh"

namespace hp {

constexpr int kK7Warps = 8;

template <int DT> struct Bits;
template <> struct Bits<HEDDLE_F32> {
  using U = uint32_t;
  __device__ static float val(U u) { return __uint_as_float(u); }
  __device__ static U top() { return 0x7F800000u; }            // +inf: "no bound"
};
template <> struct Bits<HEDDLE_U32> {
  using U = uint32_t;
  __device__ static uint32_t val(U u) { return u; }
  __device__ static U top() { return kU32Inf; }
};
template <> struct Bits<HEDDLE_F64> {
  using U = unsigned long long;
  __device__ static double val(U u) { return __longlong_as_double((long long)u); }
  __device__ static U top() { return 0x7FF0000000000000ull; }
};

template <int DT, bool KV>
struct K7Problem {
  using T = Tr<DT, HEDDLE_MINMAX>;
  using L = typename T::L;
  using G = typename T::G;
  using D = typename T::D;
  using S = typename SpT<DT>::type;
  const L* gL;
  const SolveArgs* a;
  const S* gSp;
  int b, n, m;
  // cost of items [k, e) on layer j (1-based), +inf when over the size / token caps (R6)
  __device__ D cost(int j, int k, int e) const {
    const int d = a->degrees[(int64_t)b * a->ds + j - 1];
    int row = 0;
    for (int q = 0; q < a->D; ++q) row = (a->prof_deg[q] == d) ? q : row;
    const int cap = a->caps ? a->caps[(int64_t)b * a->cs + j - 1] : -1;
    const int s = e - k;
    if (cap >= 0 && s > cap) return T::inf();
    if constexpr (KV) {
      const int64_t kvc = a->kv[(int64_t)b * a->kvs + j - 1];
      if (kvc >= 0 && gSp[e] - gSp[k] > (S)kvc) return T::inf();
    }
    const G* grow = reinterpret_cast<const G*>(a->gtab) + (int64_t)row * a->gstride;
    return T::norm(T::comb(T::zero(), gL[k], grow[s]));
  }
};

// first e in [lo, hi] with pred(e) (pred monotone false -> true); hi + 1 if none
template <class Pred>
__device__ int first_true(int lo, int hi, int lane, Pred pred) {
  while (hi - lo + 1 > 32) {
    const int step = (hi - lo + 32) / 32;
    const int e = lo + lane * step;
    const unsigned msk = __ballot_sync(0xffffffffu, e <= hi && pred(e));
    if (msk == 0) { lo = lo + min(31, (hi - lo) / step) * step + 1; continue; }   // past the last probe
    const int t = __ffs(msk) - 1;
    if (t == 0) return lo;
    const int nlo = lo + (t - 1) * step + 1;
    hi = lo + t * step;          // known true
    lo = nlo;
  }
  const int e = lo + lane;
  const unsigned msk = __ballot_sync(0xffffffffu, e <= hi && pred(e));
  return msk ? lo + __ffs(msk) - 1 : hi + 1;
}

// WPP warps per problem: 1 (many problems: one warp each) or 32 (few problems: one CTA each;
// the bisection over X becomes a 32-ary search, every warp testing one candidate per round).
template <int DT, bool KV, int WPP>
__global__ void __launch_bounds__(WPP == 1 ? 32 * kK7Warps : 32 * WPP) k7_parametric(SolveArgs a) {
  using P = K7Problem<DT, KV>;
  using T = typename P::T;
  using L = typename P::L;
  using D = typename P::D;
  using S = typename P::S;
  using U = typename Bits<DT>::U;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = WPP == 1 ? (int)(blockIdx.x * kK7Warps + warp) : (int)blockIdx.x;
  if (b >= a.B) return;
  const int m0 = prob_m(a, b), n0 = prob_n(a, b);   // ragged batches: this problem's counts
  const int m = min(max(m0, 1), a.m), n = min(max(n0, 1), a.n);
  const L* gL = reinterpret_cast<const L*>(a.lengths) + (int64_t)b * a.ls;
  __shared__ int s_err;
  __shared__ unsigned s_feas[WPP == 1 ? 1 : WPP];
  // ---- validation (same rules as the DP kernels), by the problem's first warp
  int err = 0;
  if (WPP == 1 || warp == 0) {
    for (int t = lane; t < n; t += 32) {
      const L x = gL[t];
      bool bad;
      if constexpr (DT == HEDDLE_U32) bad = (x == 0u) || (x > a.lmax_u32);
      else bad = !(x > (L)0) || !(x < (L)INFINITY);
      if (bad) err = err ? min(err, (int)HEDDLE_E_RANGE) : (int)HEDDLE_E_RANGE;
      else if (t + 1 < n && gL[t + 1] > x) err = err ? min(err, (int)HEDDLE_E_UNSORTED) : (int)HEDDLE_E_UNSORTED;
    }
    for (int j = lane; j < m; j += 32) {
      const int d = a.degrees[(int64_t)b * a.ds + j];
      int row = -1;
      for (int q = 0; q < a.D; ++q) row = (a.prof_deg[q] == d) ? q : row;
      if (row < 0) err = err ? min(err, (int)HEDDLE_E_UNKNOWN_DEGREE) : (int)HEDDLE_E_UNKNOWN_DEGREE;
      if (j + 1 < m && a.degrees[(int64_t)b * a.ds + j + 1] > d)
        err = err ? min(err, (int)HEDDLE_E_UNSORTED) : (int)HEDDLE_E_UNSORTED;
    }
    err = __reduce_min_sync(0xffffffffu, err ? err : INT_MAX);
    err = err == INT_MAX ? 0 : err;
    if (m0 != m || n0 != n) err = HEDDLE_E_INVALID;
    if (err == 0 && n < m) err = HEDDLE_E_INFEASIBLE;
  }
  S* gSp = KV ? reinterpret_cast<S*>(a.spws) + (int64_t)b * (a.n + 1) : nullptr;
  if ((WPP == 1 || warp == 0) && err == 0 && KV) {   // token prefix sums, left to right (R6)
    if (lane == 0) {
      S acc = 0;
      gSp[0] = 0;
      for (int t = 0; t < n; ++t) { acc += (S)gL[t]; gSp[t + 1] = acc; }
    }
    __syncwarp();
  }
  if constexpr (WPP > 1) {
    if (threadIdx.x == 0) s_err = err;
    __syncthreads();
    err = s_err;
  }
  P pr{gL, &a, gSp, b, n, m};
  auto feasible = [&](D X) -> bool {
    int lo = 0, hi = 0;
    for (int j = 1; j <= m; ++j) {
      if (lo + 1 > n) return false;
      if (hi >= n) {   // every end e in (lo, n] can start right after a member e-1 of R_{j-1}
        const int nlo = first_true(lo + 1, n, lane, [&](int e) { return pr.cost(j, e - 1, e) <= X; });
        if (nlo > n) return false;
        lo = nlo;      // single-item cost non-increasing in e: true from nlo to n
        continue;
      }
      if (!(pr.cost(j, hi, hi + 1) <= X)) return false;                 // R_j empty
      const int nlo = first_true(lo + 1, hi + 1, lane, [&](int e) { return pr.cost(j, e - 1, e) <= X; });
      const int nhi = first_true(hi + 1, n, lane, [&](int e) { return !(pr.cost(j, hi, e) <= X); }) - 1;
      lo = nlo;
      hi = nhi;
    }
    return lo <= n && n <= hi;
  };
  D obj = T::inf();
  if (err == 0) {
    const U top = Bits<DT>::top();
    U lo = 0, hi = top - 1;                       // smallest pattern X with feasible(X); hi: known feasible?
    bool any;
    if constexpr (WPP == 1) {
      any = feasible(Bits<DT>::val(hi));
      while (any && lo < hi) {
        const U mid = lo + (hi - lo) / 2;
        if (feasible(Bits<DT>::val(mid))) hi = mid; else lo = mid + 1;
      }
    } else {
      if (warp == 0) {
        const bool f = feasible(Bits<DT>::val(hi));
        if (lane == 0) s_feas[0] = f;
      }
      __syncthreads();
      any = s_feas[0];
      __syncthreads();
      while (any && hi - lo > 0) {                // WPP-ary search: warp w probes lo + w*step
        const U span = hi - lo;
        const U step = span / WPP + 1;
        const U x = lo + (U)warp * step;
        bool f = true;                            // probes past hi count as feasible (hi is)
        if (x < hi) f = feasible(Bits<DT>::val(x));
        if (lane == 0) s_feas[warp] = f;
        __syncthreads();
        int w = 0;
        while (w < WPP && !s_feas[w]) ++w;        // first feasible probe (monotone in X)
        __syncthreads();
        const U xw = (w < WPP) ? min(hi, lo + (U)w * step) : hi;
        const U nlo = (w == 0) ? lo : lo + (U)(w - 1) * step + 1;
        hi = xw;
        lo = min(nlo, hi);
      }
    }
    if (any) obj = Bits<DT>::val(hi);
    else err = HEDDLE_E_INFEASIBLE;
  }
  if (threadIdx.x % (WPP == 1 ? 32 : 32 * WPP) == 0) {
    a.status[b] = err;
    if (a.status_out) a.status_out[b] = err;
    reinterpret_cast<D*>(a.objective)[b] = err ? T::inf() : obj;
  }
}

}  // namespace hp
