// K10 -- short-trajectory aggregation on the device (§5.2).
//
// "Trajectories shorter than a threshold are aggregated": after the presort, the
// trajectories at or above the threshold stay single items, the shorter ones -- a suffix of the
// non-increasing order -- are cut into consecutive buckets of at most `bucket`; a bucket becomes ONE
// DP item whose length is the bucket's maximum (its first element) and whose weight is its
// cardinality, so the group size seen by F is the sum of weights (R5).  A
// threshold <= 0 is the identity.  Outputs per problem: the n' items (lengths, weights), the
// first trajectory of each item (starts, with starts[n'] = n), and n' -- a ragged batch for
// heddle_place_problem.ns.  k10_expand maps the aggregated DP's boundaries back to trajectories
// (b_j -> starts[b_j]), since items are contiguous runs of the sorted order.
#pragma once
#include <cstdint>

namespace hp {

template <class L>
__global__ void k10_aggregate(const L* __restrict__ lengths, int64_t ls, int n, double thr, int bucket,
                              L* __restrict__ agg, int32_t* __restrict__ w, int32_t* __restrict__ starts,
                              int32_t* __restrict__ n_out) {
  const int b = blockIdx.x, tid = threadIdx.x;
  const L* row = lengths + (int64_t)b * ls;
  __shared__ int s_long;
  if (tid == 0) {   // long_cnt = first index with L < thr (the row is non-increasing)
    int lo = 0, hi = n;
    if (thr > 0.0) {
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((double)row[mid] >= thr) lo = mid + 1; else hi = mid;
      }
    } else {
      lo = n;
    }
    s_long = lo;
  }
  __syncthreads();
  const int lc = s_long;
  const int np = lc + (n - lc + bucket - 1) / bucket;
  L* arow = agg + (int64_t)b * n;
  int32_t* wrow = w + (int64_t)b * n;
  int32_t* srow = starts + (int64_t)b * (n + 1);
  for (int t = tid; t < n; t += blockDim.x) {
    if (t < np) {
      const int s = t < lc ? t : lc + (t - lc) * bucket;
      const int e = t < lc ? t + 1 : min(n, s + bucket);
      arow[t] = row[s];
      wrow[t] = e - s;
      srow[t] = s;
    } else {   // padding past n' (never read: the solve uses ns)
      arow[t] = row[n - 1];
      wrow[t] = 1;
      srow[t] = n;
    }
  }
  if (tid == 0) {
    srow[n] = n;
    n_out[b] = np;
  }
}

// boundaries of the aggregated problem -> trajectory boundaries; -1 stays -1
__global__ void k10_expand(const int32_t* __restrict__ agg_b, int m, int B, const int32_t* __restrict__ starts, int n,
                           int32_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * (m + 1)) return;
  const int b = (int)(t / (m + 1));
  const int v = agg_b[t];
  out[t] = (v < 0 || v > n) ? -1 : starts[(int64_t)b * (n + 1) + v];
}

}  // namespace hp
