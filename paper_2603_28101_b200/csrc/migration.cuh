// N4 -- migration retarget (§5.3).
//
// When a trajectory's predicted length changes, the router finds its new rank among the
// n* remaining active trajectories and maps it to a worker by the plan's group sizes
// s_i scaled "proportionally to the number of remaining active trajectories": capacity
// ceil(s_i * n* / n) (R18: ceiling, so no group gets zero capacity; ranks beyond the
// scaled total go to the last worker).  One thread per query, exact int64 arithmetic.
#pragma once
#include <cstdint>

namespace hp {

__global__ void k6_retarget(const int32_t* __restrict__ bounds, int m, int B, const int32_t* __restrict__ n_active,
                            const int32_t* __restrict__ qprob, const int32_t* __restrict__ qrank, int nq,
                            int32_t* __restrict__ worker) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
    const int b = qprob[q];
    if (b < 0 || b >= B) { worker[q] = -1; continue; }
    const int32_t* bd = bounds + (int64_t)b * (m + 1);
    const int64_t n = bd[m], na = n_active[b], rank = qrank[q];
    if (n <= 0 || na < 1 || bd[0] != 0 || rank < 0 || rank >= na) { worker[q] = -1; continue; }
    int64_t cum = 0;
    int w = m - 1;                                    // overflow ranks: last worker
    for (int i = 0; i < m; ++i) {
      const int64_t s = bd[i + 1] - bd[i];
      cum += (s * na + n - 1) / n;                    // ceil(s_i * n* / n)
      if (rank < cum) { w = i; break; }
    }
    worker[q] = w;
  }
}

}  // namespace hp
