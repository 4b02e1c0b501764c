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
//  * a warp task is 64 consecutive columns: 8 column lanes x 8 columns, 4 split
//    lanes each sweeping a contiguous quarter of the split range 4 splits at a time;
//    dp[k..k+3] and L[k..k+3] are LDS.128 broadcasts, and the lane's G window slides
//    by 4 per step with one LDS.128 from the table and one from its one-shifted copy
//    (column lanes 4-7 read bank-skewed copies of both);
//  * per transition: half an FMUL2 (FMA pipe) + FMNMX (max) + half an FMNMX3 (min):
//    the ALU pipe takes 2 cycles per FMNMX and per FMNMX3 warp instruction, so a
//    warp-cell costs 3 ALU cycles -- the roofline (profiles/r01_alu_pipes_ncu.csv;
//    the FMNMX row of r01_alu_peaks.jsonl is a compiler-fusion artifact, annotated);
//  * the value pass keeps no argmin (the backtrack kernel recomputes the
//    lowest-index argmin of the m states it needs); HEDDLE_KEEP_PARENTS
//    switches to an inner loop with a strict-'<' argmin per transition;
//  * column blocks are sorted longest-first (LPT) and dealt to the warps in a static
//    snake order (HEDDLE_K2_STATIC; 0 = a shared-counter dequeue), and several CTAs
//    share an SM so one CTA's layer barrier is covered by the others.
#pragma once
#include <climits>
#include <cstdint>

#include "traits.cuh"

namespace hp {

constexpr int kLaneCols = 8;                 // columns per lane (R)
#ifndef HEDDLE_COL_LANES
#define HEDDLE_COL_LANES 8
#endif
constexpr int kColLanes = HEDDLE_COL_LANES;  // lanes across columns
constexpr int kSplitLanes = 32 / kColLanes;  // lanes across splits k, each owning a contiguous part
constexpr int kWarpCols = kColLanes * kLaneCols;   // 64 columns per warp task
constexpr int kGPad = 131;                   // G padding below s = 0; == 3 (mod 4) for LDS.128 alignment
constexpr int kGTail = kWarpCols + 8;        // G padding above s = n
constexpr int kLPad = 4 * kSplitLanes + 24;  // L / dp row padding above n (quarter rounding)
#ifndef HEDDLE_K2_UNROLL
#define HEDDLE_K2_UNROLL 4
#endif
constexpr int kK2Unroll = HEDDLE_K2_UNROLL;   // F32 min-max sweep steps per loop iteration
#ifndef HEDDLE_K2_STATIC
#define HEDDLE_K2_STATIC 1
#endif
#ifndef HEDDLE_K2_WARPS
#define HEDDLE_K2_WARPS 4
#endif
constexpr int kK2Warps = HEDDLE_K2_WARPS;
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
  const int32_t* w;        // [B][n] item weights (aggregation) or null
  int64_t ws;
  int32_t* wpws;           // [B][n+1] weight prefix sums for the backtrack (weighted mode)
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
  int* err;                // set by a dependency-wait timeout (layered kernels), or null
  int split;               // world > 1: a timeout is a peer-exchange failure (E_NCCL), else E_CUDA
  // host-input pipeline (heddle_place_solve_host): problem b's inputs are resident once
  // ready[b / ready_chunk] == ready_epoch (written by the copy engine after the chunk's copies); null: resident
  const unsigned* ready;
  unsigned ready_epoch;
  int ready_chunk;
  int vscan;               // valley kernel: descent prefixes shorter than this are scanned (K8)
  int2* rowcap;            // [B][m] {profile row, cap} per worker, written by the K3/K5 prologue, or null
  const int32_t* ms;       // [B] per-problem worker count (ragged m, <= m) or null (= m); one-CTA kernels
  const int32_t* ns;       // [B] per-problem item count (ragged n, <= n) or null (= n); one-CTA kernels
  int32_t* fbounds;        // [B][m+1] boundaries from K8's fused backtrack (every dp row kept in shared
                           // memory: small problems, few of them), or null
};

// worker count of problem b (ragged batches: SA proposals of different sizes in one launch);
// m stays the row stride of degrees / caps / boundaries and of the dp workspace
__device__ __forceinline__ int prob_m(const SolveArgs& a, int b) { return a.ms ? __ldg(a.ms + b) : a.m; }
// item count of problem b (ragged batches: e.g. aggregated problems).  n stays the
// stride of lengths / weights rows and of the per-problem workspace slabs; inside its slab a
// problem's dp rows are packed with its own stride n_b + 1 (every kernel addresses them alike)
__device__ __forceinline__ int prob_n(const SolveArgs& a, int b) { return a.ns ? __ldg(a.ns + b) : a.n; }

// counter increment with release + acquire semantics at GPU scope: the CTA's stores (ordered
// before it by a CTA barrier) are visible to whoever observes the count, and the thread that
// observes the final count sees every other CTA's stores (no separate fence.sc)
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__host__ __device__ inline int align4(int x) { return (x + 3) & ~3; }

// Debug builds (-DHEDDLE_CHECK_BOUNDS) verify, once per warp task / tile, that every shared-
// memory index the sweep will touch lies inside its array, and count violations in a device
// global (heddle_place_debug_violations()).  compute-sanitizer is not available on the pool.
#ifdef HEDDLE_CHECK_BOUNDS
__device__ unsigned long long g_hp_violations;
#define HP_CHECK(cond) do { if (!(cond)) atomicAdd(&g_hp_violations, 1ull); } while (0)
#else
#define HP_CHECK(cond) do { } while (0)
#endif

// index range touched by sweep_slide for a lane: splits [kq, kq + 4*iters) plus the prefetch of
// the window after the last step; G window indices relative to gcol: [-(k_last + 4) - 3, -kq + R]
__device__ __forceinline__ void check_sweep(int kq, int iters, int R, int sdp_lo, int sdp_hi, int g_lo, int g_hi,
                                            int gbase) {
  HP_CHECK(kq >= sdp_lo && kq + 4 * iters + 3 < sdp_hi);
  HP_CHECK(gbase - (kq + 4 * iters) - 3 >= g_lo && gbase - kq + R + 3 < g_hi);
}

// Shared-memory carve-up (bytes), identical on host and device.
template <int DT, int SR>
struct K2Smem {
  using T = Tr<DT, SR>;
  int gOff, g2Off, gbOff, g2bOff, lOff, d0Off, d1Off, kloOff, spOff, wpOff, rowOff, capOff, kvOff, total;
  __host__ __device__ K2Smem(int n, int m, bool kv, bool w = false) {
    int o = 0;
    auto take = [&](int bytes) { int at = o; o += (bytes + 15) & ~15; return at; };
    auto take128 = [&](int bytes) { o = (o + 127) & ~127; return take(bytes); };
    const int gb = (int)sizeof(typename T::G) * align4(kGPad + n + kGTail + 1);
    // two copies of the layer's cost table (and of its one-shifted copy): column lanes 0-3 read
    // copy A, lanes 4-7 copy B, whose base sits 16 bytes further in the 128-byte bank cycle.  The
    // G windows of lanes cl and cl+4 (32 columns apart = 128 bytes) then fall in different 16-byte
    // bank groups, so a warp's window loads are conflict-free (4 wavefronts, not 8).
    gOff = take128(gb);
    g2Off = take128(gb);   // sG2[t] = sG[t + 1]
    gbOff = take128(gb + 16) + 16;
    g2bOff = take128(gb + 16) + 16;
    lOff = take((int)sizeof(typename T::L) * align4(n + kLPad));
    d0Off = take((int)sizeof(typename T::D) * align4(n + kLPad));
    d1Off = take((int)sizeof(typename T::D) * align4(n + kLPad));
    kloOff = kv ? take(4 * align4(n + kLPad)) : -1;
    spOff = kv ? take(8 * (n + 1)) : -1;
    wpOff = w ? take(4 * align4(n + kLPad)) : -1;
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

// ---- F32 fast step (the paper's Eq. 3 in the default FP32 mode; min-plus uses FFMA2) -----
// Two columns share one FMUL2 (mul.rn.f32x2: L[k+u] broadcast x {G[s], G[s+1]}), so a
// cell costs 1/2 FMA-pipe issue + FMNMX(max) + 1/2 FMNMX3(min): the ALU pipe (2 cycles
// per FMNMX / FMNMX3) is the only bound.  The pair {G[x], G[x+1]} must sit in an aligned
// register pair: even x comes from the natural window, odd x from a copy of G shifted by
// one element (sG2[t] = sG[t+1]), both sliding by 4 splits per step.
__device__ __forceinline__ unsigned long long f32x2_mul_bcast(float l, unsigned long long g2) {
  unsigned long long l2, r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(l2) : "f"(l));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(l2), "l"(g2));
  return r;
}
__device__ __forceinline__ unsigned long long f32x2_fma_bcast(float l, unsigned long long g2, float d) {
  unsigned long long l2, d2, r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(l2) : "f"(l));
  asm("mov.b64 %0, {%1, %1};" : "=l"(d2) : "f"(d));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(l2), "l"(g2), "l"(d2));
  return r;
}
__device__ __forceinline__ float min3f(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ void ld2x2(const float* p, unsigned long long (&o)[2]) {
  const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(p);
  o[0] = v.x;
  o[1] = v.y;
}

// Sliding-window sweep for R columns per lane over `iters` 4-split steps starting
// at split k (a multiple of 4).  Window W[x] = G[c - k - 3 + x], x = 0..R+3; after a
// step it slides down by 4, so each step loads one LDS.128 of G (two in the F32
// min-max path: G and its shifted copy) plus the LDS.128 broadcasts of dp[k..k+3]
// and L[k..k+3].  With the loop unrolled by a multiple of the rotation period
// (R+4)/4 the window shifts compile to register renames.
template <int DT, int SR, bool KP, bool MASKED, int R>
__device__ __forceinline__ void sweep_slide(const typename Tr<DT, SR>::L* __restrict__ sL,
                                            const typename Tr<DT, SR>::D* __restrict__ sdp,
                                            const typename Tr<DT, SR>::G* __restrict__ gcol,
                                            const typename Tr<DT, SR>::G* __restrict__ gcol2, int k, int iters,
                                            typename Tr<DT, SR>::D (&acc)[R], int (&arg)[R], const int (&klo)[R]) {
  using T = Tr<DT, SR>;
  // (min-plus stays on the generic FFMA path: FFMA2 measured slower there -- its pipe, not
  //  the ALU, becomes the bound when the combine needs no FMNMX)
  if constexpr (DT == HEDDLE_F32 && SR == HEDDLE_MINMAX && !KP && !MASKED) {
    static_assert(R % 2 == 0, "column pairs");
    constexpr int P = (R + 4) / 2;          // register pairs per window
    unsigned long long wp[P], vp[P];        // wp[q] = {W[2q], W[2q+1]}, vp[q] = {W[2q+1], W[2q+2]}
    const float* gk = gcol - k - 3;
    const float* gk2 = gcol2 - k - 3;
#pragma unroll
    for (int q = 0; q < P; q += 2) {
      ld2x2(gk + 2 * q, *reinterpret_cast<unsigned long long(*)[2]>(&wp[q]));
      ld2x2(gk2 + 2 * q, *reinterpret_cast<unsigned long long(*)[2]>(&vp[q]));
    }
#pragma unroll kK2Unroll
    for (int t = 0; t < iters; ++t) {
      float dpv[4], lv[4];
      ld4(sdp + k, dpv);
      ld4(sL + k, lv);
      float v[4][R];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int r = 0; r < R; r += 2) {
          const int x = r - u + 3;           // cells (u, r), (u, r+1) use W[x], W[x+1]
          const unsigned long long g2 = (x % 2 == 0) ? wp[x / 2] : vp[(x - 1) / 2];
          if constexpr (SR == HEDDLE_MINMAX) {     // max(dp, fl(L*G)) per cell
            const unsigned long long c2 = f32x2_mul_bcast(lv[u], g2);
            float c0, c1;
            asm("mov.b64 {%0, %1}, %2;" : "=f"(c0), "=f"(c1) : "l"(c2));
            v[u][r] = fmaxf(dpv[u], c0);
            v[u][r + 1] = fmaxf(dpv[u], c1);
          } else {                                  // fma(L, G, dp): FFMA2, one rounding per cell
            const unsigned long long v2 = f32x2_fma_bcast(lv[u], g2, dpv[u]);
            asm("mov.b64 {%0, %1}, %2;" : "=f"(v[u][r]), "=f"(v[u][r + 1]) : "l"(v2));
          }
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        acc[r] = min3f(acc[r], v[0][r], v[1][r]);
        acc[r] = min3f(acc[r], v[2][r], v[3][r]);
      }
#pragma unroll
      for (int q = P - 1; q >= 2; --q) { wp[q] = wp[q - 2]; vp[q] = vp[q - 2]; }
      k += 4;
      gk -= 4;
      gk2 -= 4;
      ld2x2(gk, *reinterpret_cast<unsigned long long(*)[2]>(&wp[0]));
      ld2x2(gk2, *reinterpret_cast<unsigned long long(*)[2]>(&vp[0]));
    }
  } else {
    typename T::G w[R + 4];
    const typename T::G* gk = gcol - k - 3;
#pragma unroll
    for (int x = 0; x < R + 4; x += 4) ld4(gk + x, *reinterpret_cast<typename T::G(*)[4]>(&w[x]));
#pragma unroll 4
    for (int t = 0; t < iters; ++t) {
      typename T::D dpv[4];
      typename T::L lv[4];
      ld4(sdp + k, dpv);
      ld4(sL + k, lv);
      if constexpr (!KP) {
        // all 4R candidates first, then pairwise 3-input minima (FMNMX3 / VIMNMX3)
        typename T::D v[4][R];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int r = 0; r < R; ++r) {
            v[u][r] = T::comb(dpv[u], lv[u], w[r - u + 3]);
            if (MASKED) v[u][r] = (k + u >= klo[r]) ? v[u][r] : T::inf();
          }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          acc[r] = T::vmin(T::vmin(acc[r], v[0][r]), v[1][r]);
          acc[r] = T::vmin(T::vmin(acc[r], v[2][r]), v[3][r]);
        }
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            typename T::D v = T::comb(dpv[u], lv[u], w[r - u + 3]);
            if (MASKED) v = (k + u >= klo[r]) ? v : T::inf();
            if (v < acc[r]) { acc[r] = v; arg[r] = k + u; }   // strict '<', ascending k: lowest index
          }
        }
      }
#pragma unroll
      for (int x = R + 3; x >= 4; --x) w[x] = w[x - 4];
      k += 4;
      gk -= 4;
      ld4(gk, *reinterpret_cast<typename T::G(*)[4]>(&w[0]));
    }
  }
}

// Weighted items (short-trajectory aggregation; R5): the group size is
// Wp[i] - Wp[k], so G is gathered per cell from the worker's global cost-table row (L1-resident)
// instead of a sliding window; splits at or beyond a column give a size <= 0 (+inf).
template <int DT, int SR, bool KP, bool MASKED, int R>
__device__ __forceinline__ void sweep_weighted(const typename Tr<DT, SR>::L* __restrict__ sL,
                                               const typename Tr<DT, SR>::D* __restrict__ sdp,
                                               const int* __restrict__ sWp, const typename Tr<DT, SR>::G* __restrict__ grow,
                                               int ghi, int c, int k, int iters, int n,
                                               typename Tr<DT, SR>::D (&acc)[R], int (&arg)[R], const int (&klo)[R]) {
  using T = Tr<DT, SR>;
  int wi[R];
#pragma unroll
  for (int r = 0; r < R; ++r) wi[r] = sWp[max(0, min(c + r, n))];
#pragma unroll 2
  for (int t = 0; t < iters; ++t) {
    typename T::D dpv[4];
    typename T::L lv[4];
    int wk[4];
    ld4(sdp + k, dpv);
    ld4(sL + k, lv);
    ld4(sWp + k, wk);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int sz = wi[r] - wk[u];
        const typename T::G g = (sz >= 1 && sz <= ghi) ? __ldg(grow + sz) : T::gpad();
        typename T::D v = T::comb(dpv[u], lv[u], g);
        if (MASKED) v = (k + u >= klo[r]) ? v : T::inf();
        if (KP) {
          if (v < acc[r]) { acc[r] = v; arg[r] = k + u; }
        } else {
          acc[r] = T::vmin(acc[r], v);
        }
      }
    }
    k += 4;
  }
}

// The same with the columns' weight prefixes given (K3: the tile stages its column and split
// windows of Wp separately; sWk is indexed by the absolute split k).
template <int DT, int SR, bool KP, bool MASKED, int R>
__device__ __forceinline__ void sweep_weighted_w(const typename Tr<DT, SR>::L* __restrict__ sL,
                                                 const typename Tr<DT, SR>::D* __restrict__ sdp,
                                                 const int* __restrict__ sWk, const int (&wi)[R],
                                                 const typename Tr<DT, SR>::G* __restrict__ grow, int ghi, int k,
                                                 int iters, typename Tr<DT, SR>::D (&acc)[R], int (&arg)[R],
                                                 const int (&klo)[R]) {
  using T = Tr<DT, SR>;
#pragma unroll 2
  for (int t = 0; t < iters; ++t) {
    typename T::D dpv[4];
    typename T::L lv[4];
    int wk[4];
    ld4(sdp + k, dpv);
    ld4(sL + k, lv);
    ld4(sWk + k, wk);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int sz = wi[r] - wk[u];
        const typename T::G g = (sz >= 1 && sz <= ghi) ? __ldg(grow + sz) : T::gpad();
        typename T::D v = T::comb(dpv[u], lv[u], g);
        if (MASKED) v = (k + u >= klo[r]) ? v : T::inf();
        if (KP) {
          if (v < acc[r]) { acc[r] = v; arg[r] = k + u; }
        } else {
          acc[r] = T::vmin(acc[r], v);
        }
      }
    }
    k += 4;
  }
}

// ---------------- load + validate one problem into shared memory (K2 and K8): lengths sorted,
// finite, positive; degrees known and sorted; per-worker profile row / cap / kv cap; token and
// weight prefix sums (also written to the workspace for the backtrack).  Returns the problem's
// status; a non-zero status is already recorded (status, objective) and the CTA must return.
template <int DT, int SR, bool KV, bool W, int NT>
__device__ __forceinline__ int load_problem(const SolveArgs& a, int b, int n, int m, typename Tr<DT, SR>::L* sL,
                                            int* srow, int* scap, int64_t* skv, typename SpT<DT>::type* sSp,
                                            int* sWp, int& s_err) {
  using T = Tr<DT, SR>;
  using L = typename T::L;
  using D = typename T::D;
  using S = typename SpT<DT>::type;
  const int tid = threadIdx.x;   // n, m: this problem's item and worker counts (prob_n, prob_m)
  if (n < 1 || n > a.n) {        // ragged item count outside [1, n]
    if (tid == 0) {
      a.status[b] = HEDDLE_E_INVALID;
      if (a.status_out) a.status_out[b] = HEDDLE_E_INVALID;
      if constexpr (DT == HEDDLE_U32 && SR == HEDDLE_MINPLUS)
        reinterpret_cast<uint64_t*>(a.objective)[b] = ~0ull;
      else
        reinterpret_cast<D*>(a.objective)[b] = T::inf();
    }
    return HEDDLE_E_INVALID;
  }
  const L* gL = reinterpret_cast<const L*>(a.lengths) + (int64_t)b * a.ls;
  // ---------------- load + validate (lengths sorted/finite/positive, degrees known and sorted)
  if (tid == 0) {
    s_err = INT_MAX;
    if (a.ready) {   // wait for this problem's chunk of host inputs (copy engine, other stream)
      const unsigned* f = a.ready + b / a.ready_chunk;
      while (ld_acquire_u32(f) != a.ready_epoch) __nanosleep(256);
    }
  }
  __syncthreads();
  // inputs are read once, through L2 (ld.cg): a line shared with a neighbour problem whose chunk
  // is still in flight must not be served later from a stale L1 copy
  for (int t = tid; t < n; t += NT) sL[t] = __ldcg(gL + t);               // coalesced, batched
  for (int t = n + tid; t < align4(n + kLPad); t += NT) sL[t] = (L)1;  // finite pad: no 0*inf
  __syncthreads();
  for (int t = tid; t < n; t += NT) {
    const L x = sL[t];
    bool bad_range;
    if constexpr (DT == HEDDLE_U32) bad_range = (x == 0u) || (x > a.lmax_u32);
    else bad_range = !(x > (L)0) || !(x < (L)INFINITY);
    if (bad_range) atomicMin(&s_err, (int)HEDDLE_E_RANGE);
    else if (t + 1 < n && sL[t + 1] > x) atomicMin(&s_err, (int)HEDDLE_E_UNSORTED);
  }
  for (int j = tid; j < min(m, a.m); j += NT) {
    const int d = __ldcg(a.degrees + (int64_t)b * a.ds + j);
    int row = -1;
    for (int q = 0; q < a.D; ++q) row = (a.prof_deg[q] == d) ? q : row;
    if (row < 0) atomicMin(&s_err, (int)HEDDLE_E_UNKNOWN_DEGREE);
    if (j + 1 < min(m, a.m) && __ldcg(a.degrees + (int64_t)b * a.ds + j + 1) > d) atomicMin(&s_err, (int)HEDDLE_E_UNSORTED);
    srow[j] = row < 0 ? 0 : row;
    scap[j] = a.caps ? __ldcg(a.caps + (int64_t)b * a.cs + j) : -1;
    skv[j] = KV ? __ldcg(a.kv + (int64_t)b * a.kvs + j) : -1;
  }
  if constexpr (W) {   // weight prefix sums Wp (R5): exact, left to right; sizes must fit the cost table
    if (tid == 0) {
      int acc = 0;
      sWp[0] = 0;
      bool ok = true;
      for (int t = 0; t < n; ++t) {
        const int wt = __ldcg(a.w + (int64_t)b * a.ws + t);
        ok = ok && wt >= 1 && acc <= a.gstride - 1 - wt;
        acc += wt > 0 ? wt : 0;
        sWp[t + 1] = acc;
      }
      if (!ok) atomicMin(&s_err, (int)HEDDLE_E_RANGE);
    }
    for (int t = n + 1 + tid; t < align4(n + kLPad); t += NT) sWp[t] = INT_MAX / 2;   // beyond n: size < 0
  }
  __syncthreads();
  int err = s_err == INT_MAX ? 0 : s_err;
  if (m < 1 || m > a.m) err = HEDDLE_E_INVALID;        // ragged worker count outside [1, m]
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
    return err;
  }
  if constexpr (KV) {  // token prefix sums, left to right (R6) -- one thread, exact order
    if (tid == 0) {
      S acc = 0;
      sSp[0] = 0;
      for (int t = 0; t < n; ++t) { acc += (S)sL[t]; sSp[t + 1] = acc; }
    }
    __syncthreads();
    S* gSp = reinterpret_cast<S*>(a.spws) + (int64_t)b * (a.n + 1);   // for the backtrack
    for (int t = tid; t <= n; t += NT) gSp[t] = sSp[t];
  }
  if constexpr (W) {
    int32_t* gWp = a.wpws + (int64_t)b * (a.n + 1);   // for the backtrack
    for (int t = tid; t <= n; t += NT) gWp[t] = sWp[t];
  }
  return 0;
}

template <int DT, int SR, bool KP, bool KV, bool W = false>
#ifndef HEDDLE_K2_MINBLOCKS
#define HEDDLE_K2_MINBLOCKS 1
#endif
#ifndef HEDDLE_K2_MINMAX_BLOCKS
#define HEDDLE_K2_MINMAX_BLOCKS 4
#endif
// 32-bit min-max variants fit 128 registers without spilling: 4 CTAs (16 warps) per SM
__global__ void __launch_bounds__(kK2Threads, (SR == HEDDLE_MINMAX && DT != HEDDLE_F64) ? HEDDLE_K2_MINMAX_BLOCKS : HEDDLE_K2_MINBLOCKS)
    k2_dp_batched(SolveArgs a) {
  using T = Tr<DT, SR>;
  using L = typename T::L;
  using G = typename T::G;
  using D = typename T::D;
  using S = typename SpT<DT>::type;
  extern __shared__ __align__(16) unsigned char smem[];
  const int N = a.n, M = a.m, b = blockIdx.x;   // N, M: strides (max items / workers)
  const int n = prob_n(a, b), m = prob_m(a, b);  // this problem's
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const K2Smem<DT, SR> lay(N, M, KV, W);
  G* sG = reinterpret_cast<G*>(smem + lay.gOff);
  G* sG2 = reinterpret_cast<G*>(smem + lay.g2Off);
  G* sGb = reinterpret_cast<G*>(smem + lay.gbOff);     // bank-skewed copies (column lanes 4-7)
  G* sG2b = reinterpret_cast<G*>(smem + lay.g2bOff);
  L* sL = reinterpret_cast<L*>(smem + lay.lOff);
  D* const sdp0 = reinterpret_cast<D*>(smem + lay.d0Off);
  D* const sdp1 = reinterpret_cast<D*>(smem + lay.d1Off);
  int* sklo = KV ? reinterpret_cast<int*>(smem + lay.kloOff) : nullptr;
  S* sSp = KV ? reinterpret_cast<S*>(smem + lay.spOff) : nullptr;
  int* sWp = W ? reinterpret_cast<int*>(smem + lay.wpOff) : nullptr;
  int* srow = reinterpret_cast<int*>(smem + lay.rowOff);
  int* scap = reinterpret_cast<int*>(smem + lay.capOff);
  int64_t* skv = reinterpret_cast<int64_t*>(smem + lay.kvOff);
  __shared__ int s_err, s_ctr;
  __shared__ D s_redv[kK2Warps];
  __shared__ int s_redk[kK2Warps];

  D* gdp = reinterpret_cast<D*>(a.dpws) + (int64_t)b * (M + 1) * (N + 1);
  int32_t* gpar = KP ? a.parws + (int64_t)b * (M + 1) * (N + 1) : nullptr;
  const G* gtab = reinterpret_cast<const G*>(a.gtab);

  if (load_problem<DT, SR, KV, W, kK2Threads>(a, b, n, m, sL, srow, scap, skv, sSp, sWp, s_err) != 0) return;
  for (int t = tid; t < align4(n + kLPad); t += kK2Threads) { sdp0[t] = T::inf(); sdp1[t] = T::inf(); }

  // ---------------- layers
  for (int j = 1; j <= m; ++j) {
    D* const prev = (j & 1) ? sdp0 : sdp1;
    D* const cur = (j & 1) ? sdp1 : sdp0;
    const int imax_layer = n - m + j;                  // computed region [j, n-m+j]
    // cost table of worker j: G_j[s] for s = 1..min(n, cap), +inf padding elsewhere
    // (rebuilt only when the worker's profile row or cap changes: sorted degree
    //  vectors over a few MP degrees change row at most D-1 times per problem)
    const G* const growj = gtab + (int64_t)srow[j - 1] * a.gstride;   // weighted mode: gathered per cell
    const int ghi = (scap[j - 1] >= 0 && scap[j - 1] < a.gstride - 1) ? scap[j - 1] : a.gstride - 1;
    if (!W && (j == 1 || srow[j - 1] != srow[j - 2] || scap[j - 1] != scap[j - 2])) {
      const G* grow = gtab + (int64_t)srow[j - 1] * a.gstride;
      const int cap = scap[j - 1];
      const int hi = (cap >= 0 && cap < n) ? cap : n;
      for (int t = tid; t < kGPad + n + kGTail + 1; t += kK2Threads) {
        const int s = t - kGPad;
        const G g = (s >= 1 && s <= hi) ? grow[s] : T::gpad();
        sG[t] = g;
        sGb[t] = g;
        if (t > 0) { sG2[t - 1] = g; sG2b[t - 1] = g; }
      }
      if (tid == 0) { sG2[kGPad + n + kGTail] = T::gpad(); sG2b[kGPad + n + kGTail] = T::gpad(); }
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
        G g1;
        if constexpr (W) g1 = (sWp[i] <= ghi) ? growj[sWp[i]] : T::gpad();
        else g1 = sG[kGPad + i];
        D v = T::comb(T::zero(), sL[0], g1);
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
        G gk;
        if constexpr (W) gk = (sWp[n] - sWp[k] <= ghi) ? growj[sWp[n] - sWp[k]] : T::gpad();
        else gk = sG[kGPad + n - k];
        D v = T::comb(prev[k], sL[k], gk);
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
      // column blocks anchored at the TOP of the computed region (<= 3 surplus columns there);
      // the surplus of the partial block falls below column j, where split ranges are short
      const int ctop = align4(imax_layer - (kWarpCols - 1));
      const int nblk = (ctop + kWarpCols - 1 - j) / kWarpCols + 1;
      const int kstart = (j - 1) & ~3;
      const int cl = lane & (kColLanes - 1), kg = lane / kColLanes;
#if HEDDLE_K2_STATIC
      for (int rnd = 0;; ++rnd) {   // static snake order over the LPT-sorted blocks: no dequeue trip
        const int t = rnd * kK2Warps + ((rnd & 1) ? kK2Warps - 1 - warp : warp);
        if (rnd * kK2Warps >= nblk) break;
        if (t >= nblk) continue;
#else
      for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(&s_ctr, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= nblk) break;
#endif
        const int cb = ctop - kWarpCols * t;                  // longest block first (LPT)
        const int c = cb + kLaneCols * cl;
        const int imax = min(cb + kWarpCols - 1, imax_layer);
        const int kend = align4(imax);                       // splits k <= imax - 1
        // split-lane group kg sweeps the contiguous quarter [kstart + kg*Q, kstart + (kg+1)*Q)
        const int Q = 4 * ((kend - kstart + 4 * kSplitLanes - 1) / (4 * kSplitLanes));
        D acc[kLaneCols];
        int arg[kLaneCols], klo[kLaneCols];
#pragma unroll
        for (int r = 0; r < kLaneCols; ++r) { acc[r] = T::inf(); arg[r] = -1; klo[r] = j - 1; }
        if constexpr (KV) {
#pragma unroll
          for (int r = 0; r < kLaneCols; ++r) klo[r] = sklo[min(max(c + r, j), imax)];
        }
        if constexpr (W) {
          HP_CHECK(kstart + kg * Q >= 0 && kstart + kg * Q + Q + 3 < align4(n + kLPad));
          sweep_weighted<DT, SR, KP, KV, kLaneCols>(sL, prev, sWp, growj, ghi, c, kstart + kg * Q, Q / 4, n, acc,
                                                    arg, klo);
        } else {
          check_sweep(kstart + kg * Q, Q / 4, kLaneCols, 0, align4(n + kLPad), 0, align4(kGPad + n + kGTail + 1),
                      kGPad + c);
          const bool skew = cl >= kColLanes / 2;
          sweep_slide<DT, SR, KP, KV, kLaneCols>(sL, prev, (skew ? sGb : sG) + kGPad + c, (skew ? sG2b : sG2) + kGPad + c,
                                                 kstart + kg * Q, Q / 4,
                                                 acc, arg, klo);
        }
        // combine the kSplitLanes partial minima of each column (lowest split on ties)
#pragma unroll
        for (int off = kColLanes; off < 32; off <<= 1) {
#pragma unroll
          for (int r = 0; r < kLaneCols; ++r) {
            const D ov = __shfl_xor_sync(0xffffffffu, acc[r], off);
            if (KP) {
              const int oa = __shfl_xor_sync(0xffffffffu, arg[r], off);
              if (ov < acc[r] || (ov == acc[r] && (unsigned)oa < (unsigned)arg[r])) { acc[r] = ov; arg[r] = oa; }
            } else {
              acc[r] = T::vmin(acc[r], ov);
            }
          }
        }
        if (kg == 0) {
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
