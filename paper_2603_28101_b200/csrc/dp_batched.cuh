// K2 -- batched presorted DP, one CTA per placement problem.
//
// Computes, for every problem b of the batch and every layer j = 1..m,
//     dp[j][i] = min_{k in [j-1, i-1]} dp[j-1][k] (+) L[k] * G_j(i - k)      (Eq. 3)
// over the computed region i in [j, n-m+j] (R8), with dp[0][0] = 0
// (P:595), and writes the objective dp[m][n] (Eq. 2 makespan).
//
// B200 mapping:
//  * the whole problem lives in shared memory: L (sorted lengths), the previous
//    and current dp rows, the layer's cost table G_j[s] = T_dj * F_dj(min(s,s_max))
//    masked by the worker's cap and padded with +inf for s <= 0 (so the
//    triangular k < i bound costs no instruction) -- 17 KB at n = 1024;
//  * a warp owns 128 consecutive columns (4 per lane) and sweeps the split k
//    warp-uniformly 4 at a time: dp[k..k+3] and L[k..k+3] are LDS.128
//    broadcasts, and the lane's G window slides by 4 per step with ONE LDS.128
//    (register window of 8, unrolled x2 so no register moves);
//  * per transition: FMUL + FMNMX(max) + FMNMX(min) = 3 issue slots, the
//    measured B200 ceiling (profiles/r01_alu_peaks.jsonl: FMNMX and FMUL issue at
//    1/clk/SMSP, FMNMX3 at 1/2);
//  * the value pass keeps no argmin (the backtrack kernel recomputes the
//    lowest-index argmin of the m states it needs); HEDDLE_KEEP_PARENTS
//    switches to an inner loop with a strict-'<' argmin per transition;
//  * column blocks are handed out longest-first (LPT) through a shared counter,
//    and several CTAs share an SM so one CTA's layer barrier is covered by the others.
#pragma once
#include <climits>
#include <cstdint>

#include "traits.cuh"

namespace hp {

constexpr int kLaneCols = 4;                 // columns per lane
constexpr int kWarpCols = 32 * kLaneCols;    // columns per warp task
constexpr int kGPad = 131;                   // G padding below s = 0; == 3 (mod 4) for LDS.128 alignment
constexpr int kGTail = kWarpCols + 4;        // G padding above s = n
constexpr int kK2Warps = 4;
constexpr int kK2Threads = 32 * kK2Warps;

struct SolveArgs {
  int n, m, B;
  const void* lengths;
  int64_t ls;
  const int32_t* degrees;
  int64_t ds;
  const int32_t* caps;
  int64_t cs;
  const int64_t* kv;
  int64_t kvs;
  const void* gtab;        // [D][gstride] cost table, entry s = group size (1..max_n)
  int gstride;
  const int32_t* prof_deg; // [D] device copy of the profile's degrees
  int D;
  uint32_t lmax_u32;       // U32 range guard on lengths
  void* dpws;              // [B][m+1][n+1] dp rows for the backtrack
  int32_t* parws;          // [B][m+1][n+1] back-pointers (KEEP_PARENTS) or null
  void* spws;              // [B][n+1] token prefix sums (kv caps) or null
  int32_t* status;         // [B] workspace status
  int32_t* status_out;     // [B] caller's status or null
  void* objective;         // [B] caller's objective
};

__host__ __device__ inline int align4(int x) { return (x + 3) & ~3; }

// Shared-memory carve-up (bytes), identical on host and device.
template <int DT, int SR>
struct K2Smem {
  using T = Tr<DT, SR>;
  int gOff, lOff, d0Off, d1Off, kloOff, spOff, rowOff, capOff, kvOff, total;
  __host__ __device__ K2Smem(int n, int m, bool kv) {
    int o = 0;
    auto take = [&](int bytes) { int at = o; o += (bytes + 15) & ~15; return at; };
    gOff = take((int)sizeof(typename T::G) * align4(kGPad + n + kGTail + 1));
    lOff = take((int)sizeof(typename T::L) * align4(n + 8));
    d0Off = take((int)sizeof(typename T::D) * align4(n + 8));
    d1Off = take((int)sizeof(typename T::D) * align4(n + 8));
    kloOff = kv ? take(4 * align4(n + 8)) : -1;
    spOff = kv ? take(8 * (n + 1)) : -1;
    rowOff = take(4 * m);
    capOff = take(4 * m);
    kvOff = take(8 * m);
    total = o;
  }
};

template <class D>
__device__ __forceinline__ D shfl_down(D v, int off) { return __shfl_down_sync(0xffffffffu, v, off); }

// Sp type: exact u64 for integer lengths, FP64 otherwise (R6).
template <int DT> struct SpT { using type = double; };
template <> struct SpT<HEDDLE_U32> { using type = uint64_t; };

// One 4-split step of the warp sweep: columns c..c+3 of this lane, splits k..k+3.
// Window W[x] = G[c - k - 3 + x]: W[0..3] = lo, W[4..7] = hi.
template <int DT, int SR, bool KP, bool MASKED>
__device__ __forceinline__ void step4(const typename Tr<DT, SR>::L* __restrict__ sL,
                                      const typename Tr<DT, SR>::D* __restrict__ sdp, int k,
                                      const typename Tr<DT, SR>::G (&lo)[4],
                                      const typename Tr<DT, SR>::G (&hi)[4],
                                      typename Tr<DT, SR>::D (&acc)[kLaneCols], int (&arg)[kLaneCols],
                                      const int (&klo)[kLaneCols]) {
  using T = Tr<DT, SR>;
  typename T::D dpv[4];
  typename T::L lv[4];
  ld4(sdp + k, dpv);
  ld4(sL + k, lv);
#pragma unroll
  for (int u = 0; u < 4; ++u) {
#pragma unroll
    for (int r = 0; r < kLaneCols; ++r) {
      const int x = r - u + 3;
      const typename T::G g = x < 4 ? lo[x] : hi[x - 4];
      typename T::D v = T::comb(dpv[u], lv[u], g);
      if (MASKED) v = (k + u >= klo[r]) ? v : T::inf();
      if (KP) {
        if (v < acc[r]) { acc[r] = v; arg[r] = k + u; }   // strict '<', ascending k: lowest index
      } else {
        acc[r] = T::vmin(acc[r], v);
      }
    }
  }
}

// Sweep splits [k0, k1) (multiples of 4) for this lane's columns; gcol = sG + kGPad + c.
template <int DT, int SR, bool KP, bool MASKED>
__device__ __forceinline__ void sweep(const typename Tr<DT, SR>::L* __restrict__ sL,
                                      const typename Tr<DT, SR>::D* __restrict__ sdp,
                                      const typename Tr<DT, SR>::G* __restrict__ gcol, int k0, int k1,
                                      typename Tr<DT, SR>::D (&acc)[kLaneCols], int (&arg)[kLaneCols],
                                      const int (&klo)[kLaneCols]) {
  if (k0 >= k1) return;
  typename Tr<DT, SR>::G a[4], b[4];
  ld4(gcol - k0 - 3, a);
  ld4(gcol - k0 + 1, b);
  int k = k0;
#pragma unroll 1
  for (; k + 8 <= k1; k += 8) {
    step4<DT, SR, KP, MASKED>(sL, sdp, k, a, b, acc, arg, klo);       // window [a, b]
    ld4(gcol - k - 7, b);                                              // low part for k + 4
    step4<DT, SR, KP, MASKED>(sL, sdp, k + 4, b, a, acc, arg, klo);   // window [b, a]
    ld4(gcol - k - 11, a);                                             // low part for k + 8
  }
  if (k < k1) step4<DT, SR, KP, MASKED>(sL, sdp, k, a, b, acc, arg, klo);
}

template <int DT, int SR, bool KP, bool KV>
__global__ void __launch_bounds__(kK2Threads) k2_dp_batched(SolveArgs a) {
  using T = Tr<DT, SR>;
  using L = typename T::L;
  using G = typename T::G;
  using D = typename T::D;
  using S = typename SpT<DT>::type;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n, m = a.m, b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const K2Smem<DT, SR> lay(n, m, KV);
  G* sG = reinterpret_cast<G*>(smem + lay.gOff);
  L* sL = reinterpret_cast<L*>(smem + lay.lOff);
  D* const sdp0 = reinterpret_cast<D*>(smem + lay.d0Off);
  D* const sdp1 = reinterpret_cast<D*>(smem + lay.d1Off);
  int* sklo = KV ? reinterpret_cast<int*>(smem + lay.kloOff) : nullptr;
  S* sSp = KV ? reinterpret_cast<S*>(smem + lay.spOff) : nullptr;
  int* srow = reinterpret_cast<int*>(smem + lay.rowOff);
  int* scap = reinterpret_cast<int*>(smem + lay.capOff);
  int64_t* skv = reinterpret_cast<int64_t*>(smem + lay.kvOff);
  __shared__ int s_err, s_ctr;
  __shared__ D s_redv[kK2Warps];
  __shared__ int s_redk[kK2Warps];

  const L* gL = reinterpret_cast<const L*>(a.lengths) + (int64_t)b * a.ls;
  D* gdp = reinterpret_cast<D*>(a.dpws) + (int64_t)b * (m + 1) * (n + 1);
  int32_t* gpar = KP ? a.parws + (int64_t)b * (m + 1) * (n + 1) : nullptr;
  const G* gtab = reinterpret_cast<const G*>(a.gtab);

  // ---------------- load + validate (lengths sorted/finite/positive, degrees known and sorted)
  if (tid == 0) s_err = INT_MAX;
  __syncthreads();
  for (int t = tid; t < n; t += kK2Threads) {
    L x = gL[t];
    sL[t] = x;
    bool bad_range;
    if constexpr (DT == HEDDLE_U32) bad_range = (x == 0u) || (x > a.lmax_u32);
    else bad_range = !(x > (L)0) || !(x < (L)INFINITY);
    if (bad_range) atomicMin(&s_err, (int)HEDDLE_E_RANGE);
    else if (t + 1 < n && gL[t + 1] > x) atomicMin(&s_err, (int)HEDDLE_E_UNSORTED);
  }
  for (int t = n + tid; t < align4(n + 8); t += kK2Threads) sL[t] = (L)1;  // finite pad: no 0*inf
  for (int j = tid; j < m; j += kK2Threads) {
    const int d = a.degrees[(int64_t)b * a.ds + j];
    int row = -1;
    for (int q = 0; q < a.D; ++q) row = (a.prof_deg[q] == d) ? q : row;
    if (row < 0) atomicMin(&s_err, (int)HEDDLE_E_UNKNOWN_DEGREE);
    if (j + 1 < m && a.degrees[(int64_t)b * a.ds + j + 1] > d) atomicMin(&s_err, (int)HEDDLE_E_UNSORTED);
    srow[j] = row < 0 ? 0 : row;
    scap[j] = a.caps ? a.caps[(int64_t)b * a.cs + j] : -1;
    skv[j] = KV ? a.kv[(int64_t)b * a.kvs + j] : -1;
  }
  __syncthreads();
  int err = s_err == INT_MAX ? 0 : s_err;
  if (err == 0 && n < m) err = HEDDLE_E_INFEASIBLE;
  if (err != 0) {
    if (tid == 0) {
      a.status[b] = err;
      if (a.status_out) a.status_out[b] = err;
      if constexpr (DT == HEDDLE_U32 && SR == HEDDLE_MINPLUS)
        reinterpret_cast<uint64_t*>(a.objective)[b] = ~0ull;
      else
        reinterpret_cast<D*>(a.objective)[b] = T::inf();
    }
    return;
  }
  if constexpr (KV) {  // token prefix sums, left to right (R6) -- one thread, exact order
    if (tid == 0) {
      S acc = 0;
      sSp[0] = 0;
      for (int t = 0; t < n; ++t) { acc += (S)sL[t]; sSp[t + 1] = acc; }
    }
    __syncthreads();
    S* gSp = reinterpret_cast<S*>(a.spws) + (int64_t)b * (n + 1);   // for the backtrack
    for (int t = tid; t <= n; t += kK2Threads) gSp[t] = sSp[t];
  }
  for (int t = tid; t < align4(n + 8); t += kK2Threads) { sdp0[t] = T::inf(); sdp1[t] = T::inf(); }

  // ---------------- layers
  for (int j = 1; j <= m; ++j) {
    D* const prev = (j & 1) ? sdp0 : sdp1;
    D* const cur = (j & 1) ? sdp1 : sdp0;
    const int imax_layer = n - m + j;                  // computed region [j, n-m+j]
    // cost table of worker j: G_j[s] for s = 1..min(n, cap), +inf padding elsewhere
    {
      const G* grow = gtab + (int64_t)srow[j - 1] * a.gstride;
      const int cap = scap[j - 1];
      const int hi = (cap >= 0 && cap < n) ? cap : n;
      for (int t = tid; t < kGPad + n + kGTail + 1; t += kK2Threads) {
        const int s = t - kGPad;
        sG[t] = (s >= 1 && s <= hi) ? grow[s] : T::gpad();
      }
    }
    if constexpr (KV) {
      const int64_t kvc = skv[j - 1];
      for (int i = tid; i <= n; i += kK2Threads) {
        int lo = j - 1;
        if (kvc >= 0 && i >= j && i <= imax_layer) {
          // smallest k in [j-1, i-1] with Sp[i] - Sp[k] <= kv  (monotone in k); i if none
          int l = j - 1, h = i;
          while (l < h) {
            int mid = (l + h) >> 1;
            if (sSp[i] - sSp[mid] <= (S)kvc) h = mid; else l = mid + 1;
          }
          lo = l;
        }
        sklo[i] = lo;
      }
    }
    if (KP) {
      for (int i = tid; i <= n; i += kK2Threads)
        if (i < j || i > imax_layer) gpar[(int64_t)j * (n + 1) + i] = -1;
    }
    // entries below the computed region must read as +inf for the next layer's
    // sweep, which starts at the aligned split (j & ~3) <= j - 1 (stale values
    // from layer j-2 live there otherwise)
    if (tid < 4 && j - 1 - tid >= 0) cur[j - 1 - tid] = T::inf();
    if (tid == 0) s_ctr = 0;
    __syncthreads();

    if (j == 1) {
      // dp[1][i] = L(tau_1) * T * F(i), i in [1, n-m+1]
      for (int i = 1 + tid; i <= imax_layer; i += kK2Threads) {
        D v = T::comb(T::zero(), sL[0], sG[kGPad + i]);
        if constexpr (KV) { if (sklo[i] > 0) v = T::inf(); }
        v = T::norm(v);
        cur[i] = v;
        gdp[(int64_t)(n + 1) + i] = v;
        if (KP) gpar[(int64_t)(n + 1) + i] = (v == T::inf()) ? -1 : 0;
      }
    } else if (j == m) {
      // last layer: the single state i = n, reduced across the CTA with lowest-k ties
      const int klo0 = KV ? sklo[n] : (m - 1);
      D best = T::inf();
      int bk = INT_MAX;
      for (int k = max(m - 1, klo0) + tid; k < n; k += kK2Threads) {
        D v = T::comb(prev[k], sL[k], sG[kGPad + n - k]);
        if (v < best) { best = v; bk = k; }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        D ov = shfl_down(best, off);
        int ok = __shfl_down_sync(0xffffffffu, bk, off);
        if (ov < best || (ov == best && ok < bk)) { best = ov; bk = ok; }
      }
      if (lane == 0) { s_redv[warp] = best; s_redk[warp] = bk; }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < kK2Warps; ++w)
          if (s_redv[w] < best || (s_redv[w] == best && s_redk[w] < bk)) { best = s_redv[w]; bk = s_redk[w]; }
        D v = T::norm(best);
        cur[n] = v;
        gdp[(int64_t)m * (n + 1) + n] = v;
        if (KP) gpar[(int64_t)m * (n + 1) + n] = (v == T::inf()) ? -1 : bk;
      }
    } else {
      const int cbase = j & ~3;
      const int nblk = (imax_layer - cbase) / kWarpCols + 1;
      const int kstart = (j - 1) & ~3;
      for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(&s_ctr, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= nblk) break;
        const int cb = cbase + kWarpCols * (nblk - 1 - t);   // longest block first
        const int c = cb + kLaneCols * lane;
        const int imax = min(cb + kWarpCols - 1, imax_layer);
        const int kend = align4(imax);
        D acc[kLaneCols];
        int arg[kLaneCols], klo[kLaneCols];
#pragma unroll
        for (int r = 0; r < kLaneCols; ++r) { acc[r] = T::inf(); arg[r] = -1; klo[r] = j - 1; }
        const G* gcol = sG + kGPad + c;
        if constexpr (KV) {
#pragma unroll
          for (int r = 0; r < kLaneCols; ++r) klo[r] = sklo[min(max(c + r, j), imax)];
          const int kA = __reduce_min_sync(0xffffffffu, klo[0]);
          const int kB = __reduce_max_sync(0xffffffffu, klo[kLaneCols - 1]);
          const int ka = max(kstart, kA & ~3);
          const int kb = max(ka, min(kend, align4(kB)));
          sweep<DT, SR, KP, true>(sL, prev, gcol, ka, kb, acc, arg, klo);
          sweep<DT, SR, KP, false>(sL, prev, gcol, kb, kend, acc, arg, klo);
        } else {
          sweep<DT, SR, KP, false>(sL, prev, gcol, kstart, kend, acc, arg, klo);
        }
#pragma unroll
        for (int r = 0; r < kLaneCols; ++r) {
          const int i = c + r;
          if (i >= j && i <= imax_layer) {
            const D v = T::norm(acc[r]);
            cur[i] = v;
            gdp[(int64_t)j * (n + 1) + i] = v;
            if (KP) gpar[(int64_t)j * (n + 1) + i] = (v == T::inf()) ? -1 : arg[r];
          }
        }
      }
    }
    __syncthreads();
  }

  if (tid == 0) {
    const D obj = ((m & 1) ? sdp1 : sdp0)[n];
    const int st = (obj == T::inf()) ? (int)HEDDLE_E_INFEASIBLE : (int)HEDDLE_OK;
    a.status[b] = st;
    if (a.status_out) a.status_out[b] = st;
    if constexpr (DT == HEDDLE_U32 && SR == HEDDLE_MINPLUS)
      reinterpret_cast<uint64_t*>(a.objective)[b] = (obj == T::inf()) ? ~0ull : obj;
    else
      reinterpret_cast<D*>(a.objective)[b] = obj;
  }
}

}  // namespace hp
