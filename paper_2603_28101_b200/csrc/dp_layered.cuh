// K3 -- layered presorted DP for large n or few problems: one launch per DP layer,
// the layer's (column, split) triangle cut into uniform tiles spread over every SM.
//
// Same recurrence and arithmetic as K2 (Eq. 3; traits.cuh).  A tile is
// (problem b, 512 consecutive columns, a chunk of KC splits); the CTA stages
// dp[j-1][k0..k1), L[k0..k1) and the G window it needs (plus the one-element
// shifted copy for the FMUL2 column pairs) in shared memory, its 8 warps run the K2
// sliding sweep (64 columns each, 4 split quarters), and the per-column partial
// minima of the chunk are merged into dp[j][i] with atomicMin on the value's bit
// pattern (all values are non-negative, so the unsigned order is the value order;
// KEEP_PARENTS merges (value << 32 | k) so ties keep the lowest split).
// Persistent grid (SMs x occupancy), grid-stride over tiles.  The split mode of
// the multi-GPU driver restricts the columns a rank computes ([col_lo, col_hi)
// blocks) and exchanges finished rows between layers.
#pragma once
#include "dp_batched.cuh"

namespace hp {

constexpr int kK3Warps = 8;
constexpr int kK3Threads = 32 * kK3Warps;
constexpr int kK3Cols = kK3Warps * kWarpCols;   // 512 columns per tile
constexpr int kK3GPadLo = 23;                    // == 3 (mod 4): G staging below c0 - k1
constexpr int kK3LPad = 24;
constexpr int kK3MaxSlots = 1024;                // owned column blocks per rank (n <= 512K columns)

struct LayerArgs {
  SolveArgs a;
  int j;            // layer being computed (2..m)
  int kc;           // splits per tile (multiple of 16)
  int ncb;          // column blocks per problem
  int nq;           // split chunks per column block (max)
  int own_rank, own_world;   // split mode: compute only the column blocks zigzag-owned by own_rank
  int nown;                  // owned-block slots per rank (ncb when own_world == 1)
  const int32_t* klo;   // [B][n+1] kv lower bounds for this layer, or null
  unsigned long long* keys;   // [B][n+1] packed (value, split) minima (KEEP_PARENTS), or null
  unsigned long long* counter;   // [m+1] dynamic tile counters (zeroed per solve)
  // ---- fused NVLink exchange (split mode over peer memory) ----
  void* const* peer_dp;          // [world] every rank's dp workspace (peer pointers via CUDA IPC), or null
  unsigned long long* const* peer_flags;   // [world] every rank's arrival counters [m+1]
  unsigned long long* flags;     // this rank's arrival counters (peers add 1 per pushed block)
  unsigned int* blk_done;        // [B][ncb] finished tiles per column block of this layer (zeroed per layer)
  unsigned long long wait_prev;  // flags[j-1] target before reading row j-1 (0: no wait)
  unsigned long long wait_start; // flags[0] target before pushing into peers (solve-start barrier)
  int* err;                      // set on a spin timeout (never hang the device)
};


// Spin until *flag >= target (acquire), with a ~10 s timeout that raises *err.
__device__ __forceinline__ bool wait_flag(const unsigned long long* flag, unsigned long long target, int* err) {
  if (target == 0) return true;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= target) return true;
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 10000000000ull || *(volatile int*)err) {
      atomicExch(err, 1);
      return false;
    }
    __nanosleep(200);
  }
}

template <class D> struct AtomicBits;
template <> struct AtomicBits<float> {
  __device__ static void amin(float* p, float v) { atomicMin(reinterpret_cast<unsigned*>(p), __float_as_uint(v)); }
  __device__ static uint32_t bits(float v) { return __float_as_uint(v); }
  __device__ static float from(uint32_t b) { return __uint_as_float(b); }
};
template <> struct AtomicBits<uint32_t> {
  __device__ static void amin(uint32_t* p, uint32_t v) { atomicMin(p, v); }
  __device__ static uint32_t bits(uint32_t v) { return v; }
  __device__ static uint32_t from(uint32_t b) { return b; }
};
template <> struct AtomicBits<double> {
  __device__ static void amin(double* p, double v) {
    atomicMin(reinterpret_cast<unsigned long long*>(p), (unsigned long long)__double_as_longlong(v));
  }
};
template <> struct AtomicBits<uint64_t> {
  __device__ static void amin(uint64_t* p, uint64_t v) {
    atomicMin(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
  }
};

// ---------------------------------------------------------------- fill (+inf rows, -1 parents)
template <int DT, int SR>
__global__ void k3_fill(SolveArgs a, int64_t cells) {
  using T = Tr<DT, SR>;
  using D = typename T::D;
  D* dp = reinterpret_cast<D*>(a.dpws);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < cells; t += (int64_t)gridDim.x * blockDim.x) {
    dp[t] = T::inf();
    if (a.parws) a.parws[t] = -1;
  }
}

// ---------------------------------------------------------------- prologue: validate, Sp, layer 1
constexpr int kProThreads = 1024;
template <int DT, int SR, bool KP, bool KV>
__global__ void __launch_bounds__(kProThreads) k3_prologue(SolveArgs a) {
  using T = Tr<DT, SR>;
  using L = typename T::L;
  using G = typename T::G;
  using D = typename T::D;
  using S = typename SpT<DT>::type;
  const int n = a.n, m = a.m, b = blockIdx.x, tid = threadIdx.x;
  __shared__ int s_err;
  const L* gL = reinterpret_cast<const L*>(a.lengths) + (int64_t)b * a.ls;
  if (tid == 0) s_err = INT_MAX;
  __syncthreads();
  // U independent pairs of loads in flight per thread (one CTA per problem: a plain strided loop
  // would wait one memory round trip per element pair)
  constexpr int U = 8;
  for (int base = tid; base < n; base += U * kProThreads) {
    L x[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = min(base + u * kProThreads, n - 1);
      x[u] = gL[t];
      y[u] = gL[min(t + 1, n - 1)];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = base + u * kProThreads;
      if (t >= n) continue;
      bool bad_range;
      if constexpr (DT == HEDDLE_U32) bad_range = (x[u] == 0u) || (x[u] > a.lmax_u32);
      else bad_range = !(x[u] > (L)0) || !(x[u] < (L)INFINITY);
      if (bad_range) atomicMin(&s_err, (int)HEDDLE_E_RANGE);
      else if (t + 1 < n && y[u] > x[u]) atomicMin(&s_err, (int)HEDDLE_E_UNSORTED);
    }
  }
  int row1 = 0;
  for (int j = tid; j < m; j += blockDim.x) {
    const int d = a.degrees[(int64_t)b * a.ds + j];
    int row = -1;
    for (int q = 0; q < a.D; ++q) row = (a.prof_deg[q] == d) ? q : row;
    if (row < 0) atomicMin(&s_err, (int)HEDDLE_E_UNKNOWN_DEGREE);
    if (j + 1 < m && a.degrees[(int64_t)b * a.ds + j + 1] > d) atomicMin(&s_err, (int)HEDDLE_E_UNSORTED);
    if (a.rowcap)   // per-worker profile row and cap for K5's tiles (one load instead of three)
      a.rowcap[(int64_t)b * m + j] = make_int2(row < 0 ? 0 : row, a.caps ? a.caps[(int64_t)b * a.cs + j] : -1);
  }
  int32_t* gWp = a.w ? a.wpws + (int64_t)b * (n + 1) : nullptr;
  if (a.w && tid == 0) {   // weight prefix sums Wp (R5): exact, left to right; sizes must fit the table
    int acc = 0;
    bool ok = true;
    gWp[0] = 0;
    for (int t = 0; t < n; ++t) {
      const int wt = a.w[(int64_t)b * a.ws + t];
      ok = ok && wt >= 1 && acc <= a.gstride - 1 - wt;
      acc += wt > 0 ? wt : 0;
      gWp[t + 1] = acc;
    }
    if (!ok) atomicMin(&s_err, (int)HEDDLE_E_RANGE);
  }
  __syncthreads();
  int err = s_err == INT_MAX ? 0 : s_err;
  if (err == 0 && n < m) err = HEDDLE_E_INFEASIBLE;
  if (tid == 0) {
    a.status[b] = err;   // OK for now; the finaliser turns +inf into INFEASIBLE
    if (err != 0 && a.status_out) a.status_out[b] = err;
  }
  if (err != 0) return;
  {
    const int d = a.degrees[(int64_t)b * a.ds];
    for (int q = 0; q < a.D; ++q) row1 = (a.prof_deg[q] == d) ? q : row1;
  }
  S* gSp = KV ? reinterpret_cast<S*>(a.spws) + (int64_t)b * (n + 1) : nullptr;
  if constexpr (KV) {   // left-to-right prefix sums (R6): one thread, exact order
    if (tid == 0) {
      S acc = 0;
      gSp[0] = 0;
      for (int t = 0; t < n; ++t) { acc += (S)gL[t]; gSp[t + 1] = acc; }
    }
    __syncthreads();
  }
  // layer 1: dp[1][i] = L(tau_1) T F(i) for i in [1, n-m+1]
  const G* grow = reinterpret_cast<const G*>(a.gtab) + (int64_t)row1 * a.gstride;
  const int cap = a.caps ? a.caps[(int64_t)b * a.cs] : -1;
  const int64_t kvc = KV ? a.kv[(int64_t)b * a.kvs] : -1;
  D* gdp = reinterpret_cast<D*>(a.dpws) + (int64_t)b * (m + 1) * (n + 1);
  const L l0 = gL[0];
  const int i1 = n - m + 1;
  for (int base = 1 + tid; base <= i1; base += U * kProThreads) {
    int sz[U];
    G g[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = min(base + u * kProThreads, i1);
      sz[u] = gWp ? gWp[i] : i;   // group size of items [0, i)
    }
#pragma unroll
    for (int u = 0; u < U; ++u) g[u] = (cap >= 0 && sz[u] > cap) ? T::gpad() : grow[sz[u]];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * kProThreads;
      if (i > i1) continue;
      D v = T::comb(T::zero(), l0, g[u]);
      if constexpr (KV) { if (kvc >= 0 && gSp[i] - gSp[0] > (S)kvc) v = T::inf(); }
      v = T::norm(v);
      gdp[(int64_t)(n + 1) + i] = v;
      if (KP) a.parws[(int64_t)b * (m + 1) * (n + 1) + (n + 1) + i] = (v == T::inf()) ? -1 : 0;
    }
  }
}

// ---------------------------------------------------------------- kv lower bounds for layer j
template <int DT>
__global__ void k3_klo(SolveArgs a, int j, int32_t* klo) {
  using S = typename SpT<DT>::type;
  const int n = a.n, m = a.m;
  const int b = blockIdx.y;
  const S* gSp = reinterpret_cast<const S*>(a.spws) + (int64_t)b * (n + 1);
  const int64_t kvc = a.kv[(int64_t)b * a.kvs + j - 1];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
    int lo = j - 1;
    if (kvc >= 0 && i >= j && i <= n - m + j) {
      int l = j - 1, h = i;
      while (l < h) {
        int mid = (l + h) >> 1;
        if (gSp[i] - gSp[mid] <= (S)kvc) h = mid; else l = mid + 1;
      }
      lo = l;
    }
    klo[(int64_t)b * (n + 1) + i] = lo;
  }
}

// ---------------------------------------------------------------- split-mode column ownership
// Column blocks (kK3Cols wide, from cbase = j & ~3) are dealt to P ranks in zigzag
// order: in every group of 2P consecutive blocks rank r owns blocks r and 2P-1-r, so
// the triangular work of each pair sums to a constant (a contiguous split would leave
// the last rank 23% of the triangle at P = 8).  Slot s of rank r is its s-th block.
__host__ __device__ inline int owned_block(int slot, int rank, int world) {
  if (world <= 1) return slot;
  const int g = slot >> 1;
  return 2 * world * g + ((slot & 1) ? (2 * world - 1 - rank) : rank);
}
__host__ __device__ inline int owned_slots(int ncb, int world) {
  return world <= 1 ? ncb : 2 * ((ncb + 2 * world - 1) / (2 * world));
}

// Split-mode traffic per problem (host logic of the fused exchange): the blocks of layers 2..m
// with computed columns that `rank` owns -- each is published to the world-1 peers by the tile
// that completes it -- and the blocks owned by other ranks, whose arrival this rank waits for
// before the backtrack.  Layer m computes only column n, so only its last block counts.
__host__ inline void split_traffic(int n, int m, int world, int rank, int64_t* own, int64_t* foreign) {
  const int ncb = (n - m + 3) / kK3Cols + 1;
  *own = 0;
  *foreign = 0;
  for (int j = 2; j <= m; ++j) {
    const int cbase = j & ~3, imax = n - m + j;
    for (int blk = 0; blk < ncb; ++blk) {
      const int c0 = cbase + kK3Cols * blk;
      if (c0 > imax) break;
      if (j == m && c0 + kK3Cols <= n) continue;
      const int w = blk % (2 * world);
      if ((w < world ? w : 2 * world - 1 - w) == rank) ++*own; else ++*foreign;
    }
  }
}

// pack row j of the blocks owned by `rank` into buf[b][slot][kK3Cols] (+inf padding)
template <int DT, int SR>
__global__ void k3_pack(SolveArgs a, int j, int rank, int world, int nown, void* buf) {
  using T = Tr<DT, SR>;
  using D = typename T::D;
  const int n = a.n, m = a.m, b = blockIdx.y;
  const int cbase = j & ~3;
  const D* row = reinterpret_cast<const D*>(a.dpws) + ((int64_t)b * (m + 1) + j) * (n + 1);
  D* out = reinterpret_cast<D*>(buf) + (int64_t)b * nown * kK3Cols;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nown * kK3Cols; t += gridDim.x * blockDim.x) {
    const int i = cbase + kK3Cols * owned_block(t / kK3Cols, rank, world) + (t % kK3Cols);
    out[t] = (i <= n) ? row[i] : T::inf();
  }
}

// scatter an all-gathered buffer recv[rank][b][slot][kK3Cols] into row j of every rank's blocks
template <int DT, int SR>
__global__ void k3_unpack_rows(SolveArgs a, int j, int world, int nown, const void* recv) {
  using T = Tr<DT, SR>;
  using D = typename T::D;
  const int n = a.n, m = a.m, b = blockIdx.y;
  const int cbase = j & ~3;
  const int imax = n - m + j;
  D* row = reinterpret_cast<D*>(a.dpws) + ((int64_t)b * (m + 1) + j) * (n + 1);
  const D* in = reinterpret_cast<const D*>(recv);
  const int64_t per_rank = (int64_t)a.B * nown * kK3Cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)world * nown * kK3Cols;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(t / ((int64_t)nown * kK3Cols));
    const int rem = (int)(t % ((int64_t)nown * kK3Cols));
    const int i = cbase + kK3Cols * owned_block(rem / kK3Cols, r, world) + (rem % kK3Cols);
    if (i >= j && i <= imax) row[i] = in[r * per_rank + (int64_t)b * nown * kK3Cols + rem];
  }
}

// clear the computed region of row j to +inf (split emulation: row rebuilt from the exchange)
template <int DT, int SR>
__global__ void k3_row_fill(SolveArgs a, int j) {
  using T = Tr<DT, SR>;
  using D = typename T::D;
  const int n = a.n, m = a.m, b = blockIdx.y;
  D* row = reinterpret_cast<D*>(a.dpws) + ((int64_t)b * (m + 1) + j) * (n + 1);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x)
    if (i >= j && i <= n - m + j) row[i] = T::inf();
}

// ---------------------------------------------------------------- one layer, tiled
template <int DT, int SR>
struct K3Smem {
  using T = Tr<DT, SR>;
  int lOff, dOff, gOff, g2Off, wkOff, wcOff, total, gLen;
  __host__ __device__ K3Smem(int kc, bool w = false) {
    int o = 0;
    auto take = [&](int bytes) { int at = o; o += (bytes + 15) & ~15; return at; };
    gLen = align4(kK3Cols + kc + kK3GPadLo + 16);
    lOff = take((int)sizeof(typename T::L) * (kc + kK3LPad));
    dOff = take((int)sizeof(typename T::D) * (kc + kK3LPad));
    gOff = take((int)sizeof(typename T::G) * (gLen + 16)) + 16 * (int)sizeof(typename T::G) / 2;
    g2Off = take((int)sizeof(typename T::G) * (gLen + 16)) + 16 * (int)sizeof(typename T::G) / 2;
    wkOff = w ? take(4 * (kc + kK3LPad)) : -1;   // weight prefixes of the tile's splits (R5)
    wcOff = w ? take(4 * kK3Cols) : -1;           // and of its columns
    total = o;
  }
};

template <int DT, int SR, bool KP, bool KV, bool W = false>
__global__ void __launch_bounds__(kK3Threads) k3_layer(LayerArgs la) {
  using T = Tr<DT, SR>;
  using L = typename T::L;
  using G = typename T::G;
  using D = typename T::D;
  extern __shared__ __align__(16) unsigned char smem[];
  const SolveArgs& a = la.a;
  const int n = a.n, m = a.m, j = la.j, kc = la.kc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cl = lane & (kColLanes - 1), kg = lane / kColLanes;
  const K3Smem<DT, SR> lay(kc, W);
  L* sL = reinterpret_cast<L*>(smem + lay.lOff);
  D* sdp = reinterpret_cast<D*>(smem + lay.dOff);
  G* sG = reinterpret_cast<G*>(smem + lay.gOff);
  G* sG2 = reinterpret_cast<G*>(smem + lay.g2Off);
  int* sWk = W ? reinterpret_cast<int*>(smem + lay.wkOff) : nullptr;
  int* sWc = W ? reinterpret_cast<int*>(smem + lay.wcOff) : nullptr;
  const int imax_layer = n - m + j;
  const int cbase = j & ~3;
  const int kstart = (j - 1) & ~3;
  const int nblk = la.nown;
  // chunk counts of this rank's blocks (identical for every problem of the batch):
  // prefix s_pref over slots in descending block order (largest triangles first, LPT)
  __shared__ int s_pref[kK3MaxSlots + 1];
  __shared__ int64_t s_tile;
  if (warp == 0) {
    int carry = 0;
    for (int base = 0; base < nblk; base += 32) {
      const int sl = nblk - 1 - (base + lane);          // descending slot = descending block
      int cnt = 0;
      if (base + lane < nblk) {
        const int blk = owned_block(sl, la.own_rank, la.own_world);
        const int c0 = cbase + kK3Cols * blk;
        // (last layer: only the state i = n is on a complete partition -- R8)
        if (c0 <= imax_layer && (j < m || c0 + kK3Cols > n)) {
          const int kend = align4(min(c0 + kK3Cols - 1, imax_layer));
          cnt = (kend - kstart + kc - 1) / kc;
        }
      }
      int incl = cnt;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
      }
      if (base + lane < nblk) s_pref[base + lane + 1] = carry + incl;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_pref[0] = 0;
  }
  __syncthreads();
  const int per_prob = s_pref[nblk];
  const int64_t ntiles = (int64_t)a.B * per_prob;
  if (la.peer_dp) {   // fused exchange: row j-1 must have arrived from every peer
    __shared__ int s_ok;
    if (tid == 0) s_ok = wait_flag(la.flags + (j - 1), la.wait_prev, la.err);
    __syncthreads();
    if (!s_ok) return;
  }
  for (;;) {
    if (tid == 0) s_tile = (int64_t)atomicAdd(la.counter + j, 1ull);   // dynamic tile scheduler
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntiles) break;
    const int b = (int)(tile / per_prob);
    const int rr = (int)(tile % per_prob);
    int lo = 0, hi = nblk;                  // largest idx with s_pref[idx] <= rr
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_pref[mid] <= rr) lo = mid; else hi = mid;
    }
    const int q = rr - s_pref[lo];
    const int blk = owned_block(nblk - 1 - lo, la.own_rank, la.own_world);
    const int c0 = cbase + kK3Cols * blk;
    const int imaxb = min(c0 + kK3Cols - 1, imax_layer);
    const int kend = align4(imaxb);
    const int k0 = kstart + q * kc;
    const int k1 = min(k0 + kc, kend);
    // invalid problems compute nothing but keep the block accounting of the fused exchange
    const bool valid = a.status[b] == HEDDLE_OK;
    const L* gL = reinterpret_cast<const L*>(a.lengths) + (int64_t)b * a.ls;
    const D* gprev = reinterpret_cast<const D*>(a.dpws) + ((int64_t)b * (m + 1) + (j - 1)) * (n + 1);
    D* gcur = reinterpret_cast<D*>(a.dpws) + ((int64_t)b * (m + 1) + j) * (n + 1);
    if (valid) {
    int row = 0;
    const int d = a.degrees[(int64_t)b * a.ds + j - 1];
    for (int qq = 0; qq < a.D; ++qq) row = (a.prof_deg[qq] == d) ? qq : row;
    const G* grow = reinterpret_cast<const G*>(a.gtab) + (int64_t)row * a.gstride;
    const int cap = a.caps ? a.caps[(int64_t)b * a.cs + j - 1] : -1;
    const int ghi = (cap >= 0 && cap < n) ? cap : n;
    // ---- stage: splits [k0, k1) (+inf / 1 beyond k1 so quarter overruns contribute nothing)
    for (int t = tid; t < kc + kK3LPad; t += kK3Threads) {
      const int k = k0 + t;
      const bool in = k < k1;
      sdp[t] = in ? gprev[k] : T::inf();
      sL[t] = in ? gL[k] : (L)1;
    }
    if constexpr (W) {   // Wp of the splits (beyond k1: huge, so every size there is < 1) and columns
      const int32_t* wp = a.wpws + (int64_t)b * (n + 1);
      for (int t = tid; t < kc + kK3LPad; t += kK3Threads) sWk[t] = k0 + t < k1 ? wp[k0 + t] : INT_MAX / 2;
      for (int t = tid; t < kK3Cols; t += kK3Threads) sWc[t] = wp[min(c0 + t, n)];
    }
    // G(s) for s in [s0, s0 + gLen], s0 = c0 - k1 - kK3GPadLo (== 1 mod 4: window alignment)
    const int s0 = c0 - k1 - kK3GPadLo;
    for (int t = tid; !W && t <= lay.gLen; t += kK3Threads) {
      const int s = s0 + t;
      const G g = (s >= 1 && s <= ghi) ? grow[s] : T::gpad();
      if (t < lay.gLen) sG[t] = g;
      if (t > 0) sG2[t - 1] = g;
    }
    __syncthreads();
    // ---- sweep: warp w owns columns [c0 + 64 w, c0 + 64 w + 64)
    const int cw = c0 + kWarpCols * warp;
    if (cw <= imaxb) {
      const int c = cw + kLaneCols * cl;
      const int Q = 4 * ((k1 - k0 + 4 * kSplitLanes - 1) / (4 * kSplitLanes));
      D acc[kLaneCols];
      int arg[kLaneCols], klo[kLaneCols];
#pragma unroll
      for (int r = 0; r < kLaneCols; ++r) { acc[r] = T::inf(); arg[r] = -1; klo[r] = j - 1; }
      if constexpr (KV) {
#pragma unroll
        for (int r = 0; r < kLaneCols; ++r) klo[r] = la.klo[(int64_t)b * (n + 1) + min(max(c + r, j), imaxb)];
      }
      // shifted bases: sdpb[k] = sdp[k - k0]; gcol - k - 3 = &G(c - k - 3)
      if constexpr (W) {   // group size Wp[i] - Wp[k]: G gathered per cell from the worker's row
        const int ghi_w = (cap >= 0 && cap < a.gstride - 1) ? cap : a.gstride - 1;
        int wi[kLaneCols];
#pragma unroll
        for (int r = 0; r < kLaneCols; ++r) wi[r] = sWc[c - c0 + r];
        sweep_weighted_w<DT, SR, KP, KV, kLaneCols>(sL - k0, sdp - k0, sWk - k0, wi, grow, ghi_w, k0 + kg * Q, Q / 4,
                                                    acc, arg, klo);
      } else {
        check_sweep(k0 + kg * Q - k0, Q / 4, kLaneCols, 0, kc + kK3LPad, 0, lay.gLen, c - s0 - k0);
        sweep_slide<DT, SR, KP, KV, kLaneCols>(sL - k0, sdp - k0, sG + (c - s0), sG2 + (c - s0), k0 + kg * Q, Q / 4,
                                               acc, arg, klo);
      }
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
          if (i >= j && i <= imaxb) {
            const D v = T::norm(acc[r]);
            if constexpr (KP) {
              // (value, split) packed: lowest value, then lowest split (32-bit value types only)
              if constexpr (sizeof(D) == 4) {
                if (v != T::inf()) {
                  const unsigned long long key = ((unsigned long long)AtomicBits<D>::bits(v) << 32) | (unsigned)arg[r];
                  atomicMin(la.keys + (int64_t)b * (n + 1) + i, key);
                }
              }
            } else {
              if (v != T::inf()) AtomicBits<D>::amin(gcur + i, v);
            }
          }
        }
      }
    }
    }   // valid
    if (la.peer_dp) {
      // last finished tile of a column block pushes the block's final row values to every peer
      // over NVLink (vector stores into the peers' dp rows), then bumps their arrival counter
      __shared__ int s_last;
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        const int nch = (kend - kstart + kc - 1) / kc;
        s_last = atomicAdd(la.blk_done + (int64_t)b * la.ncb + blk, 1u) == (unsigned)(nch - 1);
        if (s_last) s_last = wait_flag(la.flags, la.wait_start, la.err);
      }
      __syncthreads();
      if (s_last) {
        __threadfence();
        const int64_t roff = ((int64_t)b * (m + 1) + j) * (n + 1);
        const D* mine = reinterpret_cast<const D*>(a.dpws) + roff;
        const int lo = max(c0, j), hi = imaxb;   // valid columns of this block
        for (int r = 0; r < la.own_world; ++r) {
          if (r == la.own_rank) continue;
          D* dst = reinterpret_cast<D*>(la.peer_dp[r]) + roff;
          for (int i = lo + tid; i <= hi; i += kK3Threads) dst[i] = ld_cg(mine + i);
        }
        __threadfence_system();
        __syncthreads();
        if (tid == 0)
          for (int r = 0; r < la.own_world; ++r)
            if (r != la.own_rank) atomicAdd_system(la.peer_flags[r] + j, 1ull);
      }
    }
    __syncthreads();   // staged rows and s_tile are reused by the next tile
  }
}

// ================================================================ K5: persistent dataflow DP
// One persistent launch computes every layer j = 2..m.  Tiles (layer, column block,
// split chunk) are dequeued in layer order from a global counter; a tile first waits
// until the blocks of row j-1 covering its split range are final (per-block "ready"
// counters, monotonic per solve), so layer j+1 starts on its low splits while layer j
// is still finishing its high columns: no per-layer launch, barrier or tail.  The
// tile that completes a column block publishes it: it bumps the block's ready counter
// and, in split mode, first stores the block's final values into every peer's dp row
// over NVLink (CUDA-IPC peer memory) and bumps the peers' counters (system scope).
// Deadlock freedom: every dependency of a tile was dequeued earlier, by a running CTA.
// Cooperative staging global -> shared with U independent loads per thread in flight before the
// stores (a plain loop issues one load, one store, one load ...: one L2 round trip per element
// row per thread).  load(t) / store(t, v) for t in [0, cnt).
template <int NT, int U, class LD, class ST>
__device__ __forceinline__ void stage_batched(int cnt, LD&& load, ST&& store) {
  for (int base = threadIdx.x; base < cnt; base += U * NT) {
    decltype(load(0)) v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = base + u * NT;
      if (t < cnt) v[u] = load(t);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = base + u * NT;
      if (t < cnt) store(t, v[u]);
    }
  }
}

struct PersistArgs {
  SolveArgs a;
  int kc, ncb;
  const int4* tiles;               // [nentries] {j, blk, q, nch(blk)}; problems interleaved b-minor
  int64_t nentries;
  unsigned long long* counter;     // global tile counter (zeroed per solve)
  int static_sched;                // 1: CTA c takes tiles c, c + grid, ... (no dequeue round trip)
  unsigned int* blk_done;          // [m+1][B][ncb] finished tiles per block (zeroed per solve)
  unsigned long long* ready;       // [m+1][B][ncb] publication counters of this rank (zeroed per solve)
  unsigned long long epoch;        // ready target (1: one publication per block per solve)
  unsigned long long* const* peer_arrive;  // split mode: every rank's total-arrivals counter
  const unsigned long long* arrive;        // this rank's total-arrivals counter (monotonic)
  unsigned long long arrive_target;        // cumulative arrivals expected at the end of this solve
  int own_rank, own_world;
  void* const* peer_dp;            // split mode: every rank's dp workspace (null: single GPU)
  unsigned long long* const* peer_ready;   // split mode: every rank's ready array
  const unsigned long long* start_flag;    // split mode: solve-start barrier counter
  unsigned long long wait_start;
  int* err;
  const int* nch;                  // [m+1][ncb] chunks per column block (single-GPU ready target)
  const void* gA;                  // cost table rows at stride gsp, row r at gA + r*gsp (16-B aligned at s == 1 mod 4)
  const void* gB;                  // the same, 16-B aligned at s == 2 mod 4 (the one-element-shifted window)
  int gsp;
  unsigned long long* trace;       // [tiles][6] %globaltimer: start, L/G staged, dependencies met, dp staged,
                                   // swept, published
                                   // (HEDDLE_PLACE_TILE_TRACE diagnostics), or null
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- 1-D bulk copies (TMA engine, cp.async.bulk) into shared memory, completed on an mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n"
               "WAIT_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
               "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// elements [t0, t1) of a staged window G(lo + t), t in [0, len), that one bulk copy from `src` (a
// cost-table row, index s) can fill: s in [1, ghi], both ends on 16-byte boundaries; empty if the
// source is not aligned there
template <class G>
__device__ __forceinline__ void bulk_span(const G* src, int lo, int len, int ghi, int& t0, int& t1) {
  constexpr int E = 16 / (int)sizeof(G);
  const int a = lo >= 1 ? lo : lo + ((1 - lo + E - 1) / E) * E;
  const int e = min(lo + len, ghi + 1);
  const int ee = e > a ? a + ((e - a) / E) * E : a;
  if (ee <= a || (reinterpret_cast<uintptr_t>(src + a) & 15)) { t0 = t1 = 0; return; }
  t0 = a - lo;
  t1 = ee - lo;
}

// Elements [t0, t1) of a staged window G(lo + t), t in [0, len), copied by ONE bulk copy rounded
// outward to 16-byte boundaries (t0 may be negative down to -(E-1), t1 may pass len by up to E-1):
// every element of the window with s in [1, ghi] comes from the copy, and those it brings in with
// s < 1 or s > ghi are overwritten with the padding after it lands (bulk_fixup).  Requires src + lo
// on a 16-byte boundary (the row-padded copies gA / gB) and smem room for the overhang.
template <class G>
__device__ __forceinline__ void bulk_span_out(int lo, int len, int ghi, int& t0, int& t1) {
  constexpr int E = 16 / (int)sizeof(G);
  const int s_lo = max(lo, 1), s_hi = min(lo + len, ghi + 1);   // needed values: s in [s_lo, s_hi)
  if (s_hi <= s_lo) { t0 = t1 = 0; return; }
  t0 = ((s_lo - lo) / E) * E;                                    // lo + t0 aligned (lo is)
  t1 = ((s_hi - lo + E - 1) / E) * E;
}

// Warp-wide spin: lane l waits until flag(l) >= target(l) (target 0: nothing to wait for), acquire
// at system scope (peers publish over NVLink) or GPU scope; ~10 s timeout raises *err.
__device__ __forceinline__ bool wait_flags_warp(const unsigned long long* flag, unsigned long long target, bool sys,
                                                int* err) {
  unsigned long long t0 = gtimer();
  for (unsigned it = 0;; ++it) {
    unsigned long long v = ~0ull;
    if (target) {
      if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
      else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    }
    if (__all_sync(0xffffffffu, v >= target)) return true;
    if ((it & 63) == 63) {   // the timeout / error word every 64 polls: one load per poll otherwise
      const bool late = gtimer() - t0 > 10000000000ull || *(volatile int*)err;
      if (__any_sync(0xffffffffu, late)) {
        if ((threadIdx.x & 31) == 0) atomicExch(err, 1);
        return false;
      }
    }
    __nanosleep(32);
  }
}

template <int DT, int SR>
__global__ void __launch_bounds__(kK3Threads, sizeof(typename Tr<DT, SR>::D) == 4 ? 3 : 2)   // 32-bit: 3 CTAs per SM, else 2
    k5_persistent(PersistArgs pa) {
  using T = Tr<DT, SR>;
  using L = typename T::L;
  using G = typename T::G;
  using D = typename T::D;
  extern __shared__ __align__(16) unsigned char smem[];
  const SolveArgs& a = pa.a;
  const int n = a.n, m = a.m, B = a.B, kc = pa.kc, ncb = pa.ncb;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cl = lane & (kColLanes - 1), kg = lane / kColLanes;
  const K3Smem<DT, SR> lay(kc);
  L* sL = reinterpret_cast<L*>(smem + lay.lOff);
  D* sdp = reinterpret_cast<D*>(smem + lay.dOff);
  G* sG = reinterpret_cast<G*>(smem + lay.gOff);
  G* sG2 = reinterpret_cast<G*>(smem + lay.g2Off);
  __shared__ int64_t s_tile;
  __shared__ int s_flag;
  __shared__ __align__(8) unsigned long long s_mbar;   // bulk-copy completion (one phase per valid tile)
  // the tile's metadata, fetched by thread 0 while the previous tile was finishing: a tile starts
  // without a dependent global load (the next tile index is dequeued at the start of the current one)
  __shared__ int4 s_tl;
  __shared__ int2 s_rc;
  __shared__ int s_valid;
  uint32_t mphase = 0;
  const int64_t ntiles = pa.nentries * B;
  auto fetch_meta = [&](int64_t t) {   // one thread
    if (t >= ntiles) return;
    const int4 q = pa.tiles[t / B];
    const int bb = (int)(t % B);
    s_tl = q;
    s_rc = a.rowcap[(int64_t)bb * m + q.x - 1];
    s_valid = a.status[bb] == HEDDLE_OK;
  };
  if (tid == 0) {
    mbar_init(&s_mbar);
    s_tile = pa.static_sched ? (int64_t)blockIdx.x : (int64_t)atomicAdd(pa.counter, 1ull);
    fetch_meta(s_tile);
  }
  for (;;) {
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntiles) break;
    unsigned long long* tr = pa.trace ? pa.trace + 6 * tile : nullptr;
    if (tr && tid == 0) tr[0] = gtimer();
    unsigned long long next = pa.static_sched ? (unsigned long long)(tile + gridDim.x) : 0ull;
    const int4 tl = s_tl;
    const int b = (int)(tile % B);
    // {j, blk | nch << 16, k0, k1}: splits [k0, k1) of column block blk (nch chunks, <= kc each)
    const int j = tl.x, blk = tl.y & 0xffff, nch = tl.y >> 16, k0 = tl.z, k1 = tl.w;
    const int imax_layer = n - m + j;
    const int cbase = j & ~3;
    const int c0 = cbase + kK3Cols * blk;
    const int imaxb = min(c0 + kK3Cols - 1, imax_layer);
    // invalid problems compute nothing but still count and publish their blocks, so that the
    // number of arrivals every rank expects does not depend on device-side validation
    const bool valid = s_valid;
    const int2 rc = s_rc;   // {profile row, cap} of worker j (prologue)
    const L* gL = reinterpret_cast<const L*>(a.lengths) + (int64_t)b * a.ls;
    const D* gprev = reinterpret_cast<const D*>(a.dpws) + ((int64_t)b * (m + 1) + (j - 1)) * (n + 1);
    D* gcur = reinterpret_cast<D*>(a.dpws) + ((int64_t)b * (m + 1) + j) * (n + 1);
    // stage only this chunk's extent (chunks on the diagonal are much shorter than kc)
    const int kl = k1 - k0;
    const int s0 = c0 - k1 - kK3GPadLo;
    const int gl = align4(kK3Cols + kl + kK3GPadLo + 16);   // == lay.gLen for a full chunk
    // ---- L and the G window do not depend on row j-1: bulk copies (TMA) of L[k0, k1), G(s0 + t)
    // and G(s0 + 1 + t) are issued by thread 0 and land while the dependency wait runs; threads
    // write only the +inf / pad elements around them
    const int cap = rc.y;
    const int ghi = (cap >= 0 && cap < n) ? cap : n;
    int a0 = 0, a1 = 0, b0 = 0, b1 = 0;
    if (valid) {
      const G* gA = reinterpret_cast<const G*>(pa.gA) + (int64_t)rc.x * pa.gsp;
      const G* gB = reinterpret_cast<const G*>(pa.gB) + (int64_t)rc.x * pa.gsp;
      // each window is one bulk copy rounded outward; outside it the window holds padding only,
      // so the threads write constants (no global loads on the tile's critical path)
      bulk_span_out<G>(s0, gl, ghi, a0, a1);
      bulk_span_out<G>(s0 + 1, gl, ghi, b0, b1);
      const bool lbulk = kl > 0 && !(reinterpret_cast<uintptr_t>(gL + k0) & 15);
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // after the last tile's generic accesses
        mbar_arrive_tx(&s_mbar, (lbulk ? kl * (uint32_t)sizeof(L) : 0u) + (uint32_t)(a1 - a0 + b1 - b0) * (uint32_t)sizeof(G));
        if (lbulk) bulk_g2s(sL, gL + k0, kl * (uint32_t)sizeof(L), &s_mbar);
        if (a1 > a0) bulk_g2s(sG + a0, gA + s0 + a0, (uint32_t)(a1 - a0) * sizeof(G), &s_mbar);
        if (b1 > b0) bulk_g2s(sG2 + b0, gB + s0 + 1 + b0, (uint32_t)(b1 - b0) * sizeof(G), &s_mbar);
      }
      for (int t = lbulk ? kl + tid : tid; t < kl + kK3LPad; t += kK3Threads) sL[t] = t < kl ? __ldg(gL + k0 + t) : (L)1;
      for (int t = tid; t < gl; t += kK3Threads) {
        if (t < a0 || t >= a1) sG[t] = T::gpad();
        if (t < b0 || t >= b1) sG2[t] = T::gpad();
      }
    }
    if (tr && tid == 0) tr[1] = gtimer();
    // ---- dependencies: row j-1 columns [max(k0, j-1), min(k1-1, n-m+j-1)] final (row 1: prologue);
    // warp 0 polls the covering blocks' counters side by side (one lane per block)
    if (warp == 0) {
      int ok = 1;
      if (valid && j >= 3) {
        const int pc = (j - 1) & ~3;
        const int lo = max(k0, j - 1), hi = min(k1 - 1, n - m + j - 1);
        const int bb1 = (hi - pc) / kK3Cols;
        for (int g = (lo - pc) / kK3Cols; ok && g <= bb1; g += 32) {
          const int bb = g + lane;
          const bool need = bb <= bb1;
          // single GPU: every chunk of a block adds 1, final at its chunk count; split: 1 per solve
          const unsigned long long target =
              !need ? 0ull : pa.peer_dp ? pa.epoch : (unsigned long long)pa.nch[(j - 1) * ncb + bb];
          ok = wait_flags_warp(pa.ready + ((int64_t)(j - 1) * B + b) * ncb + (need ? bb : 0), target,
                               pa.peer_dp != nullptr, pa.err);
        }
      }
      if (lane == 0) s_flag = ok;
    }
    __syncthreads();
    if (!s_flag) {   // timed out: let this tile's bulk copies land before the CTA exits
      if (valid) mbar_wait(&s_mbar, mphase);
      break;
    }
    if (tr && tid == 0) tr[2] = gtimer();
    if (valid) {
    mbar_wait(&s_mbar, mphase);   // the bulk copies of this tile (each thread observes completion)
    mphase ^= 1u;
    // the copies' overhang (fewer than 4 elements at each end): sizes < 1 (the triangle k >= i)
    // and over the cap become padding
    if (tid < 8) {
      const int t = tid < 4 ? a0 + tid : a1 - 8 + tid;
      if (t >= a0 && t < a1 && (s0 + t < 1 || s0 + t > ghi)) sG[t] = T::gpad();
    } else if (tid < 16) {
      const int t = tid < 12 ? b0 + tid - 8 : b1 - 16 + tid;
      if (t >= b0 && t < b1 && (s0 + 1 + t < 1 || s0 + 1 + t > ghi)) sG2[t] = T::gpad();
    }
    // row j-1 was produced by other CTAs / peers: read at L2, all loads in flight before the stores
    stage_batched<kK3Threads, sizeof(D) == 4 ? 9 : 4>(kl + kK3LPad, [&](int t) { return t < kl ? ld_cg(gprev + k0 + t) : T::inf(); },
                                 [&](int t, D v) { sdp[t] = v; });
    __syncthreads();
    if (tr && tid == 0) tr[3] = gtimer();
    const int cw = c0 + kWarpCols * warp;
    // the warp's own split range: splits at or above its top column only meet the +inf padding
    // of G (the triangle k >= i), so they are skipped -- whole warps on the diagonal chunks
    const int k1w = min(k1, align4(min(cw + kWarpCols - 1, imaxb)));
    if (cw <= imaxb && k1w > k0) {
      const int c = cw + kLaneCols * cl;
      const int Q = 4 * ((k1w - k0 + 4 * kSplitLanes - 1) / (4 * kSplitLanes));
      D acc[kLaneCols];
      int arg[kLaneCols], klo[kLaneCols];
#pragma unroll
      for (int r = 0; r < kLaneCols; ++r) { acc[r] = T::inf(); arg[r] = -1; klo[r] = j - 1; }
      check_sweep(kg * Q, Q / 4, kLaneCols, 0, kl + kK3LPad, 0, gl, c - s0 - k0);
      sweep_slide<DT, SR, false, false, kLaneCols>(sL - k0, sdp - k0, sG + (c - s0), sG2 + (c - s0), k0 + kg * Q,
                                                   Q / 4, acc, arg, klo);
#pragma unroll
      for (int off = kColLanes; off < 32; off <<= 1)
#pragma unroll
        for (int r = 0; r < kLaneCols; ++r) acc[r] = T::vmin(acc[r], __shfl_xor_sync(0xffffffffu, acc[r], off));
      if (kg == 0) {
#pragma unroll
        for (int r = 0; r < kLaneCols; ++r) {
          const int i = c + r;
          if (i >= j && i <= imaxb) {
            const D v = T::norm(acc[r]);
            if (v != T::inf()) AtomicBits<D>::amin(gcur + i, v);
          }
        }
      }
    }
    }   // valid
    // ---- completion of the column block -> publish.  The next tile is dequeued and its metadata
    // fetched here, so the round trips overlap the fence instead of starting the next iteration.
    // (Dequeuing it at the start of the current tile was measured 4 % slower on configs[4]: a
    // ready tile on the dependency chain could sit reserved behind a CTA's long current tile.)
    if (tr && tid == 0) tr[4] = gtimer();
    // the next tile's dequeue and metadata round trips (thread 32) run beside thread 0's release
    // of this one (the CTA has already read s_tile and the metadata of this tile)
    if (tid == 32) {
      if (!pa.static_sched) next = atomicAdd(pa.counter, 1ull);
      fetch_meta((int64_t)next);
      s_tile = (int64_t)next;
    }
    __syncthreads();   // the CTA's row stores precede thread 0's fence (release, cumulative)
    const int64_t bidx = ((int64_t)j * B + b) * ncb + blk;
    if (!pa.peer_dp) {   // single GPU: count the chunk; consumers wait for the block's chunk count
      if (tid == 0) {
        red_add_release_gpu(reinterpret_cast<unsigned long long*>(pa.ready + bidx), 1ull);
        if (tr) tr[5] = gtimer();
      }
      continue;
    }
    if (tid == 0) {
      // release (this chunk's stores, ordered by the barrier) + acquire (the block's other chunks)
      s_flag = atom_add_acq_rel_gpu(pa.blk_done + bidx, 1u) == (unsigned)(nch - 1);
      if (s_flag && pa.peer_dp) s_flag = wait_flag(pa.start_flag, pa.wait_start, pa.err) ? 1 : 2;
    }
    __syncthreads();
    if (s_flag) {
      if (pa.peer_dp && s_flag == 1) {
        const int64_t roff = ((int64_t)b * (m + 1) + j) * (n + 1);
        const D* mine = reinterpret_cast<const D*>(a.dpws) + roff;
        const int lo = max(c0, j), hi = imaxb;
        // 16-byte chunks (each loaded once, stored to every peer) between scalar head and tail;
        // the peers' workspaces are cudaMalloc'd like this one, so offsets align alike
        constexpr int PER = 16 / (int)sizeof(D);
        const int head = min(hi + 1 - lo, (int)((PER - (roff + lo) % PER) % PER));
        const int nvec = (hi + 1 - lo - head) / PER;
        const int vlo = lo + head, tlo = vlo + nvec * PER;
        for (int v = tid; v < nvec; v += kK3Threads) {
          const int4 x = __ldcg(reinterpret_cast<const int4*>(mine + vlo) + v);
          for (int r = 0; r < pa.own_world; ++r)
            if (r != pa.own_rank) reinterpret_cast<int4*>(reinterpret_cast<D*>(pa.peer_dp[r]) + roff + vlo)[v] = x;
        }
        for (int i = tid; i < head + (hi + 1 - tlo); i += kK3Threads) {
          const int e = i < head ? lo + i : tlo + (i - head);
          const D x = ld_cg(mine + e);
          for (int r = 0; r < pa.own_world; ++r)
            if (r != pa.own_rank) reinterpret_cast<D*>(pa.peer_dp[r])[roff + e] = x;
        }
        __syncthreads();   // every thread's peer stores precede thread 0's system fence
        if (tid == 0) {
          __threadfence_system();
          for (int r = 0; r < pa.own_world; ++r)
            if (r != pa.own_rank) {
              atomicAdd_system(pa.peer_ready[r] + bidx, 1ull);
              __threadfence_system();   // the ready increment is visible before the arrival count
              atomicAdd_system(pa.peer_arrive[r], 1ull);   // total, for the end-of-solve barrier
            }
        }
      }
      if (tid == 0) atomicAdd_system(pa.ready + bidx, 1ull);   // local consumers
    }
    if (tid == 0 && tr) tr[5] = gtimer();
  }
}

#ifndef HEDDLE_INST_TU   // non-template kernels: defined in heddle_place.cu's translation unit only
// split mode: wait until every block the peers publish in this solve has arrived (all rows
// complete for the backtrack, and no push is still in flight when the next solve resets)
__global__ void k5_wait_arrivals(PersistArgs pa) {
  wait_flag(pa.arrive, pa.arrive_target, pa.err);
  __threadfence();
}

// ---------------------------------------------------------------- fused exchange helpers
// solve-start barrier: announce to every peer that this rank's workspace is reset
__global__ void k3_signal_start(unsigned long long* const* peer_flags, int rank, int world) {
  __threadfence_system();
  for (int r = 0; r < world; ++r)
    if (r != rank) atomicAdd_system(peer_flags[r], 1ull);
}
// wait for the last layer's blocks from every peer before finalising / backtracking
__global__ void k3_wait(const unsigned long long* flag, unsigned long long target, int* err) {
  wait_flag(flag, target, err);
  __threadfence();
}
#endif

// ---------------------------------------------------------------- KEEP_PARENTS: unpack keys of layer j
template <int DT, int SR>
__global__ void k3_unpack(SolveArgs a, int j, unsigned long long* keys) {
  using T = Tr<DT, SR>;
  using D = typename T::D;
  const int n = a.n, m = a.m, b = blockIdx.y;
  if constexpr (sizeof(D) == 4) {
    D* gcur = reinterpret_cast<D*>(a.dpws) + ((int64_t)b * (m + 1) + j) * (n + 1);
    int32_t* pcur = a.parws + ((int64_t)b * (m + 1) + j) * (n + 1);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
      unsigned long long& key = keys[(int64_t)b * (n + 1) + i];
      if (key != ~0ull) {
        gcur[i] = AtomicBits<D>::from((uint32_t)(key >> 32));
        pcur[i] = (int32_t)(key & 0xffffffffu);
      }
      key = ~0ull;
    }
  }
}

// ---------------------------------------------------------------- finaliser
template <int DT, int SR>
__global__ void k3_finalize(SolveArgs a) {
  using T = Tr<DT, SR>;
  using D = typename T::D;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  const int n = a.n, m = a.m;
  if (a.err && *(volatile int*)a.err)   // a dependency wait timed out: the rows are incomplete
    a.status[b] = a.split ? HEDDLE_E_NCCL : HEDDLE_E_CUDA;
  if (a.status[b] != HEDDLE_OK) {
    if (a.status_out) a.status_out[b] = a.status[b];
    if constexpr (DT == HEDDLE_U32 && SR == HEDDLE_MINPLUS) reinterpret_cast<uint64_t*>(a.objective)[b] = ~0ull;
    else reinterpret_cast<D*>(a.objective)[b] = T::inf();
    return;
  }
  const D obj = reinterpret_cast<const D*>(a.dpws)[((int64_t)b * (m + 1) + m) * (n + 1) + n];
  const int st = (obj == T::inf()) ? (int)HEDDLE_E_INFEASIBLE : (int)HEDDLE_OK;
  a.status[b] = st;
  if (a.status_out) a.status_out[b] = st;
  if constexpr (DT == HEDDLE_U32 && SR == HEDDLE_MINPLUS)
    reinterpret_cast<uint64_t*>(a.objective)[b] = (obj == T::inf()) ? ~0ull : obj;
  else
    reinterpret_cast<D*>(a.objective)[b] = obj;
}

}  // namespace hp
