// C-ABI of the B200-native presorted-DP placement (include/heddle_place.h).
// Host side: argument validation, profile validation, workspace, kernel
// dispatch.  Device side: K1 cost tables (this file), K2 batched DP
// (dp_batched.cuh), K4 backtrack (backtrack.cuh).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <new>
#include <string>
#include <vector>
#include <algorithm>

#include "aggregate.cuh"
#include "anneal.cuh"
#include "backtrack.cuh"
#include "dp_batched.cuh"
#include "dp_layered.cuh"
#include "dispatch.h"
#include "heddle_place.h"
#include "migration.cuh"
#include "parametric.cuh"
#include "valley.cuh"

using namespace hp;

// ------------------------------------------------------------------------ K1
// Cost tables G_d[s] = T_d * F_d(min(s, s_max)) for s = 1..max_n (
// clamp S:90).  Entry 0 is never read.  F32: fl32(T*F); F64: T*F; U32: exact.
template <int DT>
__global__ void k1_cost_tables(const void* T, const void* F, int D, int s_max, int gstride, void* gtab) {
  const int d = blockIdx.y;
  for (int s = 1 + blockIdx.x * blockDim.x + threadIdx.x; s < gstride; s += gridDim.x * blockDim.x) {
    const int f = (s < s_max ? s : s_max) - 1;
    if constexpr (DT == HEDDLE_F32) {
      reinterpret_cast<float*>(gtab)[(int64_t)d * gstride + s] =
          __fmul_rn(reinterpret_cast<const float*>(T)[d], reinterpret_cast<const float*>(F)[(int64_t)d * s_max + f]);
    } else if constexpr (DT == HEDDLE_F64) {
      reinterpret_cast<double*>(gtab)[(int64_t)d * gstride + s] =
          __dmul_rn(reinterpret_cast<const double*>(T)[d], reinterpret_cast<const double*>(F)[(int64_t)d * s_max + f]);
    } else {
      reinterpret_cast<uint32_t*>(gtab)[(int64_t)d * gstride + s] =
          reinterpret_cast<const uint32_t*>(T)[d] * reinterpret_cast<const uint32_t*>(F)[(int64_t)d * s_max + f];
    }
  }
}

// ------------------------------------------------------------------------ context
// solve_host input pipeline: about kPipeChunks chunks of at least kPipeMinChunk problems
constexpr int64_t kPipeChunks = 16;
constexpr int64_t kPipeMinChunk = 256;

struct heddle_place_ctx {
  int device = 0, dtype = 0, semiring = 0;
  int max_n = 0, max_m = 0, max_batch = 0, D = 0, s_max = 0;
  uint32_t flags = 0;
  int gstride = 0;
  uint32_t lmax_u32 = 0;
  void* d_gtab = nullptr;
  int32_t* d_prof_deg = nullptr;
  void* d_dp = nullptr;
  int32_t* d_par = nullptr;
  void* d_sp = nullptr;
  int32_t* d_status = nullptr;
  void* d_stage = nullptr;
  size_t stage_bytes = 0;
  cudaStream_t copy_stream = nullptr;   // solve_host input pipeline: copy stream, its last event,
  cudaEvent_t copy_done = nullptr;      // per-chunk ready flags (device) and the call epoch (pinned host)
  unsigned* d_chunk_ready = nullptr;
  unsigned* h_epoch = nullptr;
  unsigned pipe_epoch = 0;
  bool solved = false;
  bool last_kv = false;
  SolveArgs last{};
  int64_t launches = 0;
  int smem_optin = 0;
  int k2_smem_max = 0;
  int k8_smem_max = 0;
  ValleyWs vws{};                       // K8L range-minimum workspace (allocated on first use)
  int num_sms = 0;
  int32_t* d_klo = nullptr;             // [max_batch][max_n+1] (layered kernel, kv caps)
  int32_t* d_wp = nullptr;              // [max_batch][max_n+1] weight prefix sums (weighted problems)
  bool last_w = false;
  unsigned long long* d_keys = nullptr; // [max_batch][max_n+1] (layered kernel, KEEP_PARENTS)
  unsigned long long* d_ctr = nullptr;  // [max_m+1] dynamic tile counters of the layered kernel
  bool last_layered = false;
  // split mode (one large instance over several GPUs)
  int split_rank = 0, split_world = 1;
  bool split_emulate = false;           // all virtual ranks on this device, exchange by copy (tests)
  ncclComm_t comm = nullptr;
  void* d_send = nullptr;
  void* d_recv = nullptr;
  size_t xbuf_bytes = 0;
  // tracing (HEDDLE_PLACE_TRACE=1): per-phase device time of the layered path, printed per solve
  bool trace = false;
  // fused NVLink exchange (split mode): peers' dp workspaces and arrival counters via CUDA IPC
  bool p2p = false;
  void** d_peer_dp = nullptr;                 // device array [world]
  unsigned long long** d_peer_flags = nullptr; // device array [world]
  unsigned long long* d_flags = nullptr;      // [max_m+1] this rank's arrival counters (monotonic)
  std::vector<void*> peer_dp_h, peer_flags_h; // opened IPC mappings (host copies, for cleanup)
  unsigned int* d_blkdone = nullptr;          // [max_batch][ncb_max]
  int* d_err = nullptr;
  int64_t epoch = 0;                          // collective solves so far (same on every rank)
  // persistent dataflow kernel (K5)
  unsigned long long* d_ready = nullptr;      // [max_m+1][max_batch][ncb_max] per-block epoch counters
  unsigned long long** d_peer_ready = nullptr; // device array [world]
  std::vector<void*> peer_ready_h;
  int4* d_tiles = nullptr;
  int* d_nch = nullptr;                      // [m+1][ncb] chunks per column block of the cached tile list
  int2* d_rowcap = nullptr;                   // [max_batch][max_m] {profile row, cap} (K3/K5 prologue)
  void* d_gpad = nullptr;                     // K5 TMA staging: two row-padded copies of the cost table
  int gsp = 0;                                //   (row stride gsp; copy A offset 3, copy B offset 2 elements)
  size_t tiles_cap = 0;
  int64_t tiles_n = 0;
  int tiles_key[7] = {-1, -1, -1, -1, -1, -1, -1};
  int64_t ready_epoch = 0;                    // solves that used d_ready (single-GPU and split)
  unsigned long long arrive_total = 0;        // cumulative K5 arrivals expected (split mode)
  unsigned long long** d_peer_arrive = nullptr; // device array [world]: &peer_flags[r][max_m + 1]
  std::vector<unsigned long long> expect;     // cumulative arrivals expected per counter
  // device-resident annealer (K9, heddle_place_anneal): chain state, proposals, solver outputs
  void* d_sa = nullptr;
  size_t sa_bytes = 0;
  cudaStream_t sa_stream = nullptr;           // capture stream of the per-iteration CUDA graph
  std::vector<int> prof_degrees;              // host copy of the profile's degrees
  int32_t* d_fbounds = nullptr;               // [max_batch][max_m+1] K8 fused-backtrack boundaries
  bool last_fused = false;
};

namespace {

size_t elem_size(int dtype) { return dtype == HEDDLE_F64 ? 8 : 4; }   // lengths / profile / cost table
size_t dp_elem_size(int dtype, int semiring) {
  return (dtype == HEDDLE_F64 || dtype == HEDDLE_F32X || (dtype == HEDDLE_U32 && semiring == HEDDLE_MINPLUS)) ? 8 : 4;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

template <int DT, int SR> int k3_smem_t(int kc, bool w) { return K3Smem<DT, SR>(kc, w).total; }
int k3_smem(int dt, int sr, int kc, bool w = false) { return HP_DISPATCH(k3_smem_t, kc, w); }

int k2_smem(int dt, int sr, int n, int m, bool kv, bool w = false) {
  if (dt == HEDDLE_F32X) return K2Smem<HEDDLE_F32X, HEDDLE_MINPLUS>(n, m, kv, w).total;
  if (dt == HEDDLE_F32) return sr == HEDDLE_MINMAX ? K2Smem<HEDDLE_F32, HEDDLE_MINMAX>(n, m, kv, w).total : K2Smem<HEDDLE_F32, HEDDLE_MINPLUS>(n, m, kv, w).total;
  if (dt == HEDDLE_F64) return sr == HEDDLE_MINMAX ? K2Smem<HEDDLE_F64, HEDDLE_MINMAX>(n, m, kv, w).total : K2Smem<HEDDLE_F64, HEDDLE_MINPLUS>(n, m, kv, w).total;
  return sr == HEDDLE_MINMAX ? K2Smem<HEDDLE_U32, HEDDLE_MINMAX>(n, m, kv, w).total : K2Smem<HEDDLE_U32, HEDDLE_MINPLUS>(n, m, kv, w).total;
}

// K8 / K8L (valley solver, min-max only)
int k8_smem(int dt, int n, int m, bool kv, bool w) {
  if (dt == HEDDLE_F32) return K8Smem<HEDDLE_F32>(n, m, kv, w).total;
  if (dt == HEDDLE_F64) return K8Smem<HEDDLE_F64>(n, m, kv, w).total;
  return K8Smem<HEDDLE_U32>(n, m, kv, w).total;
}

template <int DT, int SR>
int fill_launch(const SolveArgs& a, int64_t cells, int grid, cudaStream_t s) {
  k3_fill<DT, SR><<<grid, 256, 0, s>>>(a, cells);
  return 0;
}
template <int DT, int SR>
int klo_launch(const SolveArgs& a, int j, int32_t* klo, dim3 g, cudaStream_t s) {
  k3_klo<DT><<<g, 256, 0, s>>>(a, j, klo);
  return 0;
}
template <int DT, int SR>
int unpack_launch(const SolveArgs& a, int j, unsigned long long* keys, dim3 g, cudaStream_t s) {
  k3_unpack<DT, SR><<<g, 256, 0, s>>>(a, j, keys);
  return 0;
}
template <int DT, int SR>
int pack_launch(const SolveArgs& a, int j, int rank, int world, int nown, void* buf, dim3 g, cudaStream_t s) {
  k3_pack<DT, SR><<<g, 256, 0, s>>>(a, j, rank, world, nown, buf);
  return 0;
}
template <int DT, int SR>
int unpack_rows_launch(const SolveArgs& a, int j, int world, int nown, const void* recv, dim3 g, cudaStream_t s) {
  k3_unpack_rows<DT, SR><<<g, 256, 0, s>>>(a, j, world, nown, recv);
  return 0;
}
template <int DT, int SR>
int row_fill_launch(const SolveArgs& a, int j, dim3 g, cudaStream_t s) {
  k3_row_fill<DT, SR><<<g, 256, 0, s>>>(a, j);
  return 0;
}
template <int DT, int SR>
int finalize_launch(const SolveArgs& a, cudaStream_t s) {
  k3_finalize<DT, SR><<<(a.B + 255) / 256, 256, 0, s>>>(a);
  return 0;
}

template <class V>
bool check_profile(const heddle_place_config* c, double* gmax) {
  const V* T = static_cast<const V*>(c->T);
  const V* F = static_cast<const V*>(c->F);
  *gmax = 0;
  for (int d = 0; d < c->num_degrees; ++d) {
    const double t = (double)T[d];
    if (!(t > 0) || !std::isfinite(t)) return false;
    for (int s = 0; s < c->s_max; ++s) {
      const double f = (double)F[(int64_t)d * c->s_max + s];
      if (!(f > 0) || !std::isfinite(f)) return false;
      if (s > 0 && f < (double)F[(int64_t)d * c->s_max + s - 1]) return false;   // premise P:560
    }
    const double g = t * (double)F[(int64_t)d * c->s_max + c->s_max - 1];
    if (g > *gmax) *gmax = g;
  }
  return true;
}


// Batched (one CTA per problem) vs layered (all SMs per layer) -- rough cost model:
// batched: waves x per-problem cells / (~12 cells/clk for one 4-warp CTA);
// layered: all cells / (~30 cells/clk/SM x SMs) + per-layer launch/drain (~6000 clk).
// layered (persistent dataflow): max(all cells / (~30 cells/clk/SM x SMs), critical path of m dependent
// tiles of 512 columns x kc splits at ~11 cells/clk) -- see k5_kc().
int k5_kc(int n, int m, int B, int num_sms, int world = 1) {
  const double cells = (double)B * (double)heddle_place_transitions(n, m) / world;   // this rank's share
  const double work = cells / (30.0 * num_sms);
  int kc = 2048;
  while (kc > 256 && (double)m * kK3Cols * std::min(kc, n) / 11.0 > 0.25 * work) kc /= 2;
  return kc;
}
bool use_layered(const heddle_place_ctx* x, int n, int m, int B) {
  const double cells = (double)heddle_place_transitions(n, m);
  const double slots = (double)x->num_sms * 8.0;
  const double waves = std::ceil((double)B / slots);
  const double t2 = waves * cells / 12.0;
  const int kc = k5_kc(n, m, B, x->num_sms);
  const double t3 = std::max((double)B * cells / (30.0 * x->num_sms), (double)m * kK3Cols * std::min(kc, n) / 11.0) +
                    20000.0;
  return t3 < t2;
}

// Does the one-CTA-per-problem kernel (K2, or K8 with HEDDLE_VALLEY) serve this solve?  (Only
// those kernels can take pipelined host inputs, see heddle_place_solve_host.)
bool per_problem_kernel(const heddle_place_ctx* x, int n, int m, int B, bool kv, bool wt) {
  if (x->split_world > 1) return false;
  if (x->flags & HEDDLE_VALLEY)   // K8 whenever the problem fits shared memory, else K8L
    return !(x->flags & HEDDLE_FORCE_LAYERED) && k8_smem(x->dtype, n, m, kv, wt) <= x->k8_smem_max;
  if (x->flags & HEDDLE_FORCE_BATCHED) return true;
  if (x->flags & HEDDLE_FORCE_LAYERED) return false;
  return k2_smem(x->dtype, x->semiring, n, m, kv, wt) <= x->k2_smem_max && !use_layered(x, n, m, B);
}

// K5 (persistent dataflow over all layers); fill + prologue have been enqueued already.
heddle_status solve_persistent(heddle_place_ctx* x, SolveArgs& a, cudaStream_t s) {
  const int dt = x->dtype, sr = x->semiring;
  const int n = a.n, m = a.m, B = a.B, world = x->split_world, rank = x->split_rank;
  int kc = k5_kc(n, m, B, x->num_sms, world);
  // throughput-bound solves (the chain allows chunks of >= 512 splits): twice the chunk at 2
  // resident CTAs per SM instead of 3 -- measured 3.8 / 3.4 / 6.2 % faster on the large instance
  // at 1 / 2 / 4 GPUs (profiles/r01_k5_variants.jsonl); latency-bound solves keep 3 CTAs per SM
  const bool big_tiles = kc >= 512;
  if (big_tiles) kc *= 2;
  if (const char* e = std::getenv("HEDDLE_PLACE_K5_KC")) kc = std::max(64, std::atoi(e) & ~15);   // tuning
  const int ncb = (n - m + 3) / kK3Cols + 1;
  const int ncb_max = (x->max_n + 3) / kK3Cols + 2;
  if (!x->d_ready) {
    const size_t bytes = 8 * (size_t)(x->max_m + 1) * x->max_batch * ncb_max;
    if (cudaMalloc(&x->d_ready, bytes) != cudaSuccess || cudaMemset(x->d_ready, 0, bytes) != cudaSuccess) {
      cudaGetLastError();
      return HEDDLE_E_NOMEM;
    }
  }
  if (!x->d_blkdone) {
    if (cudaMalloc(&x->d_blkdone, sizeof(unsigned) * (size_t)x->max_batch * ncb_max * (x->max_m + 1)) != cudaSuccess) {
      cudaGetLastError();
      return HEDDLE_E_NOMEM;
    }
  }
  if (!x->d_err) {
    if (cudaMalloc(&x->d_err, sizeof(int)) != cudaSuccess || cudaMemset(x->d_err, 0, sizeof(int)) != cudaSuccess) {
      cudaGetLastError();
      return HEDDLE_E_NOMEM;
    }
  }
  // tile list (layer-major; inside a layer ascending first split, then block; this rank's blocks
  // only), cached per shape.  A block's splits [kstart, kend) are cut into chunks of kc, except the
  // diagonal part [c0 - 4, kend): it reads row j-1's block of the same index -- the last one that
  // layer finishes -- so it forms the dependency chain through the layers and is cut into small
  // chunks of kd splits that run side by side on different SMs.
  int kd = kc;   // (measured: small diagonal chunks did not shorten the solve, profiles/r01_k5_variants.jsonl)
  if (const char* e = std::getenv("HEDDLE_PLACE_K5_KD")) kd = std::max(16, std::min(kc, std::atoi(e) & ~3));
  const int key[7] = {n, m, kc, rank, world, ncb, kd};
  if (std::memcmp(key, x->tiles_key, sizeof(key)) != 0) {
    std::vector<int4> tl;
    const int nown = owned_slots(ncb, world);
    for (int j = 2; j <= m; ++j) {
      const int cbase = j & ~3, kstart = (j - 1) & ~3, imax = n - m + j;
      std::vector<int4> lt;   // {k0, blk, k1, nch}
      for (int sl = 0; sl < nown; ++sl) {
        const int blk = owned_block(sl, rank, world);
        const int c0 = cbase + kK3Cols * blk;
        if (blk >= ncb || c0 > imax || (j == m && c0 + kK3Cols <= n)) continue;
        const int kend = align4(std::min(c0 + kK3Cols - 1, imax));
        const int tlo = kd < kc ? std::min(kend, std::max(kstart, c0 - 4)) : kend;
        std::vector<std::pair<int, int>> ch;
        for (int k0 = kstart; k0 < tlo; k0 += kc) ch.push_back({k0, std::min(k0 + kc, tlo)});
        for (int k0 = tlo; k0 < kend; k0 += kd) ch.push_back({k0, std::min(k0 + kd, kend)});
        for (auto& c : ch) lt.push_back(make_int4(c.first, blk, c.second, (int)ch.size()));
      }
      std::sort(lt.begin(), lt.end(), [](const int4& p, const int4& q) {
        return p.x != q.x ? p.x < q.x : p.y < q.y;
      });
      for (auto& t : lt) tl.push_back(make_int4(j, t.y | (t.w << 16), t.x, t.z));
    }
    if (tl.size() > x->tiles_cap) {
      cudaFree(x->d_tiles);
      x->d_tiles = nullptr;
      x->tiles_cap = 0;
      if (cudaMalloc(&x->d_tiles, sizeof(int4) * tl.size()) != cudaSuccess) { cudaGetLastError(); return HEDDLE_E_NOMEM; }
      x->tiles_cap = tl.size();
    }
    if (!tl.empty() && cudaMemcpy(x->d_tiles, tl.data(), sizeof(int4) * tl.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      return HEDDLE_E_CUDA;
    std::vector<int> nchv((size_t)(m + 1) * ncb, 0);   // chunks per (layer, block)
    for (auto& t : tl) nchv[(size_t)t.x * ncb + (t.y & 0xffff)] = t.y >> 16;
    cudaFree(x->d_nch);
    x->d_nch = nullptr;
    if (cudaMalloc(&x->d_nch, sizeof(int) * nchv.size()) != cudaSuccess) { cudaGetLastError(); return HEDDLE_E_NOMEM; }
    if (cudaMemcpy(x->d_nch, nchv.data(), sizeof(int) * nchv.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      return HEDDLE_E_CUDA;
    x->tiles_n = (int64_t)tl.size();
    std::memcpy(x->tiles_key, key, sizeof(key));
  }
  x->ready_epoch++;
  // per-solve reset (safe in split mode: peers publish into this rank only after its start
  // signal, and the previous solve waited for all of its arrivals)
  if (cudaMemsetAsync(x->d_ctr, 0, 8, s) != cudaSuccess ||
      cudaMemsetAsync(x->d_blkdone, 0, sizeof(unsigned) * (size_t)B * ncb * (m + 1), s) != cudaSuccess ||
      cudaMemsetAsync(x->d_ready, 0, 8 * (size_t)B * ncb * (m + 1), s) != cudaSuccess ||
      cudaMemsetAsync(x->d_err, 0, sizeof(int), s) != cudaSuccess)
    return HEDDLE_E_CUDA;
  // cost-table copies for the bulk (TMA) staging of G windows: rows padded to a multiple of 4
  // elements, copy A shifted by 3 and copy B by 2, so the windows K5 stages (start == 1 mod 4,
  // and the one-element-shifted copy) begin on 16-byte boundaries
  if (!x->d_gpad) {
    const size_t es = elem_size(dt);
    x->gsp = align4(x->gstride) + 4;
    const size_t half = (size_t)x->D * x->gsp + 4;
    if (cudaMalloc(&x->d_gpad, 2 * es * half) != cudaSuccess) { cudaGetLastError(); return HEDDLE_E_NOMEM; }
    for (int c = 0; c < 2; ++c) {
      char* dst = static_cast<char*>(x->d_gpad) + es * (c * half + (c == 0 ? 3 : 2));
      if (cudaMemcpy2DAsync(dst, es * x->gsp, x->d_gtab, es * x->gstride, es * x->gstride, x->D,
                            cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return HEDDLE_E_CUDA;
    }
  }
  PersistArgs pa{};
  {
    const size_t es = elem_size(dt), half = (size_t)x->D * x->gsp + 4;
    pa.gA = static_cast<char*>(x->d_gpad) + es * 3;
    pa.gB = static_cast<char*>(x->d_gpad) + es * (half + 2);
    pa.gsp = x->gsp;
  }
  pa.a = a;
  pa.kc = kc;
  pa.ncb = ncb;
  pa.tiles = x->d_tiles;
  pa.nch = x->d_nch;
  pa.nentries = x->tiles_n;
  pa.counter = x->d_ctr;
  if (const char* e = std::getenv("HEDDLE_PLACE_K5_STATIC")) pa.static_sched = std::atoi(e);   // A/B
  pa.blk_done = x->d_blkdone;
  pa.ready = x->d_ready;
  pa.epoch = 1ull;
  pa.own_rank = rank;
  pa.own_world = world;
  pa.err = x->d_err;
  pa.a.err = x->d_err;   // a dependency-wait timeout becomes an error status, not a silent partial row
  a.err = x->d_err;
  pa.a.split = a.split = world > 1;
  if (world > 1) {
    x->epoch++;
    if ((int)x->expect.size() < x->max_m + 1) x->expect.assign(x->max_m + 1, 0ull);
    x->expect[0] += (unsigned long long)(world - 1);
    k3_signal_start<<<1, 1, 0, s>>>(x->d_peer_flags, rank, world);
    x->launches++;
    pa.peer_dp = x->d_peer_dp;
    pa.peer_ready = x->d_peer_ready;
    pa.start_flag = x->d_flags;
    pa.wait_start = x->expect[0];
    // arrivals: one per (problem, block of layers 2..m with computed columns) owned by another rank
    int64_t own = 0, foreign = 0;
    split_traffic(n, m, world, rank, &own, &foreign);
    x->arrive_total += (unsigned long long)foreign * B;
    pa.peer_arrive = x->d_peer_arrive;
    pa.arrive = x->d_flags + x->max_m + 1;
    pa.arrive_target = x->arrive_total;
  }
  K5Fn fn = k5_for(dt, sr);
  const int smem = k3_smem(dt, sr, kc);
  int occ = 0;
  cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kK3Threads, smem);
  if (occ < 1) return HEDDLE_E_CUDA;
  const int64_t ntiles = x->tiles_n * B;
  // resident CTAs per SM: 3 for latency-bound solves, 2 with the doubled chunks (more CTAs stretch
  // every tile and with it the dependency chain through the layers)
  int per_sm = std::min(occ, big_tiles ? 2 : 3);
  if (const char* e = std::getenv("HEDDLE_PLACE_K5_CTAS")) per_sm = std::max(1, std::min(occ, std::atoi(e)));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)per_sm * x->num_sms));
  std::vector<cudaEvent_t> tev(2);
  if (x->trace) {
    for (auto& e : tev) cudaEventCreate(&e);
    cudaEventRecord(tev[0], s);
  }
  // HEDDLE_PLACE_TILE_TRACE=<file>: append this solve's per-tile timeline (diagnostics only)
  const char* ttrace = std::getenv("HEDDLE_PLACE_TILE_TRACE");
  unsigned long long* d_trace = nullptr;
  if (ttrace && ttrace[0]) {
    if (cudaMalloc(&d_trace, 48 * (size_t)ntiles) != cudaSuccess) { cudaGetLastError(); d_trace = nullptr; }
    else cudaMemsetAsync(d_trace, 0, 48 * (size_t)ntiles, s);
    pa.trace = d_trace;
  }
  fn<<<grid, kK3Threads, smem, s>>>(pa);
  x->launches++;
  if (d_trace) {
    std::vector<unsigned long long> h(6 * (size_t)ntiles);
    std::vector<int4> tl(x->tiles_n);
    cudaMemcpyAsync(h.data(), d_trace, 48 * (size_t)ntiles, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(tl.data(), x->d_tiles, sizeof(int4) * tl.size(), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    cudaFree(d_trace);
    const std::string tpath = world > 1 ? std::string(ttrace) + ".r" + std::to_string(rank) : std::string(ttrace);
    if (FILE* f = std::fopen(tpath.c_str(), "ab")) {   // record: int64 {ntiles, B, kc, grid, rank, world}, int4 tiles, u64 times
      const int64_t hdr[6] = {ntiles, B, kc, grid, rank, world};
      std::fwrite(hdr, sizeof(hdr), 1, f);
      std::fwrite(tl.data(), sizeof(int4), tl.size(), f);
      std::fwrite(h.data(), 8, h.size(), f);
      std::fclose(f);
    }
  }
  if (world > 1) {
    k5_wait_arrivals<<<1, 1, 0, s>>>(pa);
    x->launches++;
  }
  if (x->trace) {
    cudaEventRecord(tev[1], s);
    cudaStreamSynchronize(s);
    float ms = 0;
    cudaEventElapsedTime(&ms, tev[0], tev[1]);
    std::fprintf(stderr, "[heddle_place trace] persistent rank %d/%d n=%d m=%d B=%d kc=%d grid=%d tiles=%lld: %.3f ms\n",
                 rank, world, n, m, B, kc, grid, (long long)ntiles, ms);
    for (auto& e : tev) cudaEventDestroy(e);
  }
  HP_DISPATCH(finalize_launch, a, s);
  x->launches++;
  return cudaGetLastError() == cudaSuccess ? HEDDLE_OK : HEDDLE_E_CUDA;
}

heddle_status solve_layered(heddle_place_ctx* x, SolveArgs& a, bool kp, bool kv, cudaStream_t s) {
  const int dt = x->dtype, sr = x->semiring;
  const int n = a.n, m = a.m, B = a.B;
  // workspace of the layered path (allocated on first use)
  if (kv && !x->d_klo) {
    if (cudaMalloc(&x->d_klo, 4 * (size_t)x->max_batch * (x->max_n + 1)) != cudaSuccess) { cudaGetLastError(); return HEDDLE_E_NOMEM; }
  }
  if (kp && !x->d_keys) {
    if (cudaMalloc(&x->d_keys, 8 * (size_t)x->max_batch * (x->max_n + 1)) != cudaSuccess) { cudaGetLastError(); return HEDDLE_E_NOMEM; }
    if (cudaMemsetAsync(x->d_keys, 0xff, 8 * (size_t)x->max_batch * (x->max_n + 1), s) != cudaSuccess) return HEDDLE_E_CUDA;
  }
  if (!x->d_ctr) {
    if (cudaMalloc(&x->d_ctr, 8 * (size_t)(x->max_m + 1)) != cudaSuccess) { cudaGetLastError(); return HEDDLE_E_NOMEM; }
  }
  if (cudaMemsetAsync(x->d_ctr, 0, 8 * (size_t)(m + 1), s) != cudaSuccess) return HEDDLE_E_CUDA;
  if (!x->d_rowcap) {
    if (cudaMalloc(&x->d_rowcap, sizeof(int2) * (size_t)x->max_batch * x->max_m) != cudaSuccess) { cudaGetLastError(); return HEDDLE_E_NOMEM; }
  }
  a.rowcap = x->d_rowcap;
  const int64_t cells = (int64_t)B * (m + 1) * (n + 1);
  const int fill_grid = (int)std::min<int64_t>((cells + 255) / 256, (int64_t)x->num_sms * 16);
  HP_DISPATCH(fill_launch, a, cells, fill_grid, s);
  pro_for(dt, sr, kp, kv)<<<B, kProThreads, 0, s>>>(a);
  x->launches += 2;
  const bool wt = a.w != nullptr;   // aggregation weights (R5): the prologue wrote Wp; K3 only
  const char* nok5 = std::getenv("HEDDLE_PLACE_NO_PERSISTENT");
  if (!kp && !kv && !wt && !(x->split_world > 1 && (x->split_emulate || !x->p2p)) && !(nok5 && nok5[0] == '1'))
    return solve_persistent(x, a, s);
  // tile geometry: 256 columns x kc splits; kc sized for >= ~4 tiles per resident CTA
  // (per rank in split mode: each rank computes 1/world of the layer's cells)
  const double layer_cells = (double)B * (double)(n - m + 1) * (double)(n - m + 2) / 2.0 / x->split_world;
  K3Fn fn = k3_for(dt, sr, kp, kv, wt);
  int kc = 2048;
  int occ = 0;
  for (;;) {
    const int sm = k3_smem(dt, sr, kc, wt);
    cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kK3Threads, sm);
    const double tiles = layer_cells / ((double)kK3Cols * kc);
    if (kc <= 256 || tiles >= 4.0 * occ * x->num_sms) break;
    kc /= 2;
  }
  if (occ < 1) return HEDDLE_E_CUDA;
  const int smem = k3_smem(dt, sr, kc, wt);
  LayerArgs la{};
  la.a = a;
  la.kc = kc;
  la.ncb = (n - m + 3) / kK3Cols + 1;
  la.nq = (n + 3) / kc + 1;
  const int world = x->split_world;
  la.own_world = world;
  la.own_rank = x->split_rank;
  la.nown = owned_slots(la.ncb, world);
  la.klo = kv ? x->d_klo : nullptr;
  la.keys = kp ? x->d_keys : nullptr;
  la.counter = x->d_ctr;
  if (la.nown > kK3MaxSlots) return HEDDLE_E_INVALID;
  const int64_t ntiles = (int64_t)B * la.nown * la.nq;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)occ * x->num_sms);
  // split-mode exchange buffers: send [B][nown][kK3Cols], recv [world][B][nown][kK3Cols]
  const size_t des = dp_elem_size(dt, sr);
  const size_t slab = (size_t)B * la.nown * kK3Cols;
  if (world > 1 && x->xbuf_bytes < slab * des) {
    cudaFree(x->d_send);
    cudaFree(x->d_recv);
    x->d_send = x->d_recv = nullptr;
    x->xbuf_bytes = 0;
    if (cudaMalloc(&x->d_send, slab * des) != cudaSuccess || cudaMalloc(&x->d_recv, slab * des * world) != cudaSuccess) {
      cudaGetLastError();
      return HEDDLE_E_NOMEM;
    }
    x->xbuf_bytes = slab * des;
  }
  const ncclDataType_t nt = dt == HEDDLE_F32 ? ncclFloat32 : (dt == HEDDLE_F64 || dt == HEDDLE_F32X) ? ncclFloat64
                            : (sr == HEDDLE_MINMAX ? ncclUint32 : ncclUint64);
  const dim3 pg((unsigned)std::min<int64_t>((slab / B + 255) / 256, 1024), B);
  const dim3 ug((unsigned)std::min<int64_t>((slab * world / B + 255) / 256, 2048), B);
  std::vector<cudaEvent_t> tev;
  if (x->trace) {
    tev.resize(3 * (size_t)m);
    for (auto& e : tev) cudaEventCreate(&e);
  }
  const bool p2p = world > 1 && x->p2p && !x->split_emulate;
  if (p2p) {
    // fused NVLink exchange: counters are monotonic across solves; expected arrivals are
    // accumulated per layer (blocks with computed columns owned by the other ranks)
    x->epoch++;
    if ((int)x->expect.size() < x->max_m + 1) x->expect.assign(x->max_m + 1, 0ull);
    x->expect[0] += (unsigned long long)(world - 1);
    if (cudaMemsetAsync(x->d_blkdone, 0, sizeof(unsigned) * (size_t)B * la.ncb * (m + 1), s) != cudaSuccess)
      return HEDDLE_E_CUDA;
    k3_signal_start<<<1, 1, 0, s>>>(x->d_peer_flags, x->split_rank, world);
    x->launches++;
    la.peer_dp = x->d_peer_dp;
    la.peer_flags = x->d_peer_flags;
    la.flags = x->d_flags;
    la.err = x->d_err;
    la.a.err = x->d_err;
    la.a.split = 1;
    la.wait_start = x->expect[0];
  }
  for (int j = 2; j <= m; ++j) {
    la.j = j;
    if (kv) {
      dim3 g((n + 256) / 256, B);
      HP_DISPATCH(klo_launch, a, j, x->d_klo, g, s);
      x->launches++;
    }
    if (p2p) {
      la.blk_done = x->d_blkdone + (size_t)B * la.ncb * j;
      la.wait_prev = j >= 3 ? x->expect[j - 1] : 0ull;
      // arrivals for row j: one per (problem, block with computed columns) owned by another rank
      const int cbase = j & ~3, imax = n - m + j;
      int foreign = 0;
      for (int blk = 0; blk < la.ncb; ++blk) {
        if (cbase + kK3Cols * blk > imax) break;
        const int w = blk % (2 * world);
        const int owner = w < world ? w : 2 * world - 1 - w;   // inverse of owned_block()
        if (owner != x->split_rank) ++foreign;
      }
      x->expect[j] += (unsigned long long)foreign * B;
    }
    if (x->trace) cudaEventRecord(tev[3 * j - 6], s);
    if (world > 1 && x->split_emulate) {
      // every virtual rank computes its blocks; the all-gather is emulated by packing each
      // rank's blocks into its recv slab, clearing the row and unpacking it again
      for (int vr = 0; vr < world; ++vr) {
        la.own_rank = vr;
        if (cudaMemsetAsync(x->d_ctr + j, 0, 8, s) != cudaSuccess) return HEDDLE_E_CUDA;
        fn<<<grid, kK3Threads, smem, s>>>(la);
        x->launches++;
      }
      for (int vr = 0; vr < world; ++vr) {
        HP_DISPATCH(pack_launch, a, j, vr, world, la.nown, static_cast<char*>(x->d_recv) + vr * slab * des, pg, s);
        x->launches++;
      }
      HP_DISPATCH(row_fill_launch, a, j, dim3((n + 256) / 256, B), s);
      HP_DISPATCH(unpack_rows_launch, a, j, world, la.nown, x->d_recv, ug, s);
      x->launches += 2;
    } else {
      fn<<<grid, kK3Threads, smem, s>>>(la);
      x->launches++;
      if (x->trace) cudaEventRecord(tev[3 * j - 5], s);
      if (world > 1 && !p2p) {
        HP_DISPATCH(pack_launch, a, j, x->split_rank, world, la.nown, x->d_send, pg, s);
        if (ncclAllGather(x->d_send, x->d_recv, slab, nt, x->comm, s) != ncclSuccess) return HEDDLE_E_NCCL;
        HP_DISPATCH(unpack_rows_launch, a, j, world, la.nown, x->d_recv, ug, s);
        x->launches += 2;
      }
    }
    if (x->trace) cudaEventRecord(tev[3 * j - 4], s);
    if (kp) {
      dim3 g((n + 256) / 256, B);
      HP_DISPATCH(unpack_launch, a, j, x->d_keys, g, s);
      x->launches++;
    }
  }
  if (p2p) {   // the last row must have arrived before the finaliser and the backtrack read it
    k3_wait<<<1, 1, 0, s>>>(x->d_flags + m, m >= 2 ? x->expect[m] : 0ull, x->d_err);
    x->launches++;
  }
  if (x->trace) {
    cudaStreamSynchronize(s);
    float tk = 0, tx = 0, ms = 0, mx = 0;
    for (int j = 2; j <= m; ++j) {
      cudaEventElapsedTime(&ms, tev[3 * j - 6], tev[3 * j - 5]);
      tk += ms;
      cudaEventElapsedTime(&ms, tev[3 * j - 5], tev[3 * j - 4]);
      tx += ms;
      mx = ms > mx ? ms : mx;
    }
    std::fprintf(stderr, "[heddle_place trace] rank %d/%d n=%d m=%d B=%d kc=%d grid=%d: layer kernels %.3f ms, "
                 "exchange %.3f ms (max %.1f us/layer)\n", x->split_rank, world, n, m, B, kc, grid, tk, tx, 1e3 * mx);
    for (auto& e : tev) cudaEventDestroy(e);
  }
  if (p2p) { a.err = x->d_err; a.split = 1; }
  HP_DISPATCH(finalize_launch, a, s);
  x->launches++;
  return cudaGetLastError() == cudaSuccess ? HEDDLE_OK : HEDDLE_E_CUDA;
}

}  // namespace

extern "C" {

const char* heddle_place_strerror(heddle_status s) {
  switch (s) {
    case HEDDLE_OK: return "ok";
    case HEDDLE_E_INVALID: return "invalid argument";
    case HEDDLE_E_UNSORTED: return "lengths or degrees not sorted non-increasing";
    case HEDDLE_E_INFEASIBLE: return "infeasible (n < m or capacities cannot cover n)";
    case HEDDLE_E_RANGE: return "value out of range (NaN/inf/<=0, F decreasing, or U32 overflow guard)";
    case HEDDLE_E_UNKNOWN_DEGREE: return "MP degree not in the profile";
    case HEDDLE_E_STATE: return "bad call order or missing HEDDLE_KEEP_PARENTS";
    case HEDDLE_E_CUDA: return "CUDA error";
    case HEDDLE_E_NCCL: return "NCCL error";
    case HEDDLE_E_NOMEM: return "out of memory";
  }
  return "unknown status";
}

int64_t heddle_place_transitions(int32_t n, int32_t m) {
  if (n < 1 || m < 1 || n < m) return 0;
  if (m == 1) return 1;
  const int64_t w = (int64_t)n - m + 1;
  return 2 * w + (int64_t)(m - 2) * w * (w + 1) / 2;
}

int64_t heddle_place_launch_count(const heddle_place_ctx* ctx) { return ctx ? ctx->launches : -1; }

void heddle_place_destroy(heddle_place_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard g(ctx->device);
  cudaFree(ctx->d_gtab);
  cudaFree(ctx->d_prof_deg);
  cudaFree(ctx->d_dp);
  cudaFree(ctx->d_par);
  cudaFree(ctx->d_sp);
  cudaFree(ctx->d_status);
  cudaFree(ctx->d_stage);
  cudaFree(ctx->d_sa);
  cudaFree(ctx->d_fbounds);
  if (ctx->sa_stream) cudaStreamDestroy(ctx->sa_stream);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->copy_done) cudaEventDestroy(ctx->copy_done);
  cudaFree(ctx->d_chunk_ready);
  cudaFree(ctx->vws.mask);
  cudaFree(ctx->vws.bm);
  cudaFree(ctx->vws.sp);
  cudaFree(ctx->vws.smd);
  cudaFree(ctx->vws.dlast);
  cudaFree(ctx->vws.dlrun);
  cudaFree(ctx->vws.done);
  cudaFree(ctx->vws.khint);
  if (ctx->h_epoch) cudaFreeHost(ctx->h_epoch);
  cudaFree(ctx->d_klo);
  cudaFree(ctx->d_wp);
  cudaFree(ctx->d_keys);
  cudaFree(ctx->d_ctr);
  cudaFree(ctx->d_send);
  cudaFree(ctx->d_recv);
  for (size_t r = 0; r < ctx->peer_dp_h.size(); ++r)
    if ((int)r != ctx->split_rank && ctx->peer_dp_h[r]) cudaIpcCloseMemHandle(ctx->peer_dp_h[r]);
  for (size_t r = 0; r < ctx->peer_flags_h.size(); ++r)
    if ((int)r != ctx->split_rank && ctx->peer_flags_h[r]) cudaIpcCloseMemHandle(ctx->peer_flags_h[r]);
  for (size_t r = 0; r < ctx->peer_ready_h.size(); ++r)
    if ((int)r != ctx->split_rank && ctx->peer_ready_h[r]) cudaIpcCloseMemHandle(ctx->peer_ready_h[r]);
  cudaFree(ctx->d_peer_dp);
  cudaFree(ctx->d_peer_flags);
  cudaFree(ctx->d_peer_ready);
  cudaFree(ctx->d_peer_arrive);
  cudaFree(ctx->d_ready);
  cudaFree(ctx->d_tiles);
  cudaFree(ctx->d_nch);
  cudaFree(ctx->d_rowcap);
  cudaFree(ctx->d_gpad);
  cudaFree(ctx->d_flags);
  cudaFree(ctx->d_blkdone);
  cudaFree(ctx->d_err);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  delete ctx;
}

heddle_status heddle_place_init(const heddle_place_config* c, heddle_place_ctx** out) {
  if (!out) return HEDDLE_E_INVALID;
  *out = nullptr;
  if (!c || !c->degrees || !c->T || !c->F) return HEDDLE_E_INVALID;
  if (c->dtype < HEDDLE_U32 || c->dtype > HEDDLE_F32X) return HEDDLE_E_INVALID;
  if (c->dtype == HEDDLE_F32X && c->semiring != HEDDLE_MINPLUS) return HEDDLE_E_INVALID;   // nothing to accumulate
  if (c->semiring != HEDDLE_MINMAX && c->semiring != HEDDLE_MINPLUS) return HEDDLE_E_INVALID;
  if ((c->flags & HEDDLE_VALLEY) && c->semiring != HEDDLE_MINMAX) return HEDDLE_E_INVALID;   // no valley in a sum
  if (c->max_n < 1 || c->max_m < 1 || c->max_batch < 1 || c->num_degrees < 1 || c->s_max < 1) return HEDDLE_E_INVALID;
  if (c->max_n > (1 << 24)) return HEDDLE_E_INVALID;
  for (int d = 0; d < c->num_degrees; ++d) {
    if (c->degrees[d] <= 0) return HEDDLE_E_INVALID;
    for (int e = 0; e < d; ++e)
      if (c->degrees[e] == c->degrees[d]) return HEDDLE_E_INVALID;
  }
  double gmax = 0;
  uint32_t lmax = 0;
  if (c->dtype == HEDDLE_F32 || c->dtype == HEDDLE_F32X) {
    if (!check_profile<float>(c, &gmax)) return HEDDLE_E_RANGE;
  } else if (c->dtype == HEDDLE_F64) {
    if (!check_profile<double>(c, &gmax)) return HEDDLE_E_RANGE;
  } else {
    if (!check_profile<uint32_t>(c, &gmax)) return HEDDLE_E_RANGE;
    const uint32_t* T = static_cast<const uint32_t*>(c->T);
    const uint32_t* F = static_cast<const uint32_t*>(c->F);
    uint64_t g64 = 0;
    for (int d = 0; d < c->num_degrees; ++d) {
      const uint64_t g = (uint64_t)T[d] * (uint64_t)F[(int64_t)d * c->s_max + c->s_max - 1];
      if (g > g64) g64 = g;
    }
    if (g64 >= (uint64_t)kU32Thresh) return HEDDLE_E_RANGE;
    // every admissible cost L*G must stay below 2^32 - 65536 and L <= 65535 (traits.cuh)
    const uint64_t lim = ((uint64_t)kU32Thresh - 1) / g64;
    lmax = (uint32_t)(lim < 65535 ? lim : 65535);
    if (lmax < 1) return HEDDLE_E_RANGE;
  }

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || c->device < 0 || c->device >= ndev) return HEDDLE_E_CUDA;
  DeviceGuard guard(c->device);
  heddle_place_ctx* x = new (std::nothrow) heddle_place_ctx();
  if (!x) return HEDDLE_E_NOMEM;
  x->device = c->device;
  x->dtype = c->dtype;
  x->semiring = c->semiring;
  x->max_n = c->max_n;
  x->max_m = c->max_m;
  x->max_batch = c->max_batch;
  x->D = c->num_degrees;
  x->prof_degrees.assign(c->degrees, c->degrees + c->num_degrees);
  x->s_max = c->s_max;
  x->flags = c->flags;
  x->gstride = c->max_n + 1;
  x->lmax_u32 = lmax;
  {
    const char* tr = std::getenv("HEDDLE_PLACE_TRACE");
    x->trace = tr && tr[0] == '1';
  }
  cudaDeviceGetAttribute(&x->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
  cudaDeviceGetAttribute(&x->num_sms, cudaDevAttrMultiProcessorCount, c->device);

  const size_t es = elem_size(c->dtype);
  const size_t des = dp_elem_size(c->dtype, c->semiring);
  const size_t cells = (size_t)c->max_batch * (size_t)(c->max_m + 1) * (size_t)(c->max_n + 1);
  void *dT = nullptr, *dF = nullptr;
  bool ok = cudaMalloc(&x->d_gtab, es * (size_t)x->D * x->gstride) == cudaSuccess &&
            cudaMalloc(&x->d_prof_deg, 4 * (size_t)x->D) == cudaSuccess &&
            cudaMalloc(&x->d_dp, des * cells) == cudaSuccess &&
            cudaMalloc(&x->d_sp, 8 * (size_t)c->max_batch * (size_t)(c->max_n + 1)) == cudaSuccess &&
            cudaMalloc(&x->d_status, 4 * (size_t)c->max_batch) == cudaSuccess &&
            cudaMalloc(&dT, es * (size_t)x->D) == cudaSuccess &&
            cudaMalloc(&dF, es * (size_t)x->D * c->s_max) == cudaSuccess;
  if (ok && (c->flags & HEDDLE_KEEP_PARENTS)) ok = cudaMalloc(&x->d_par, 4 * cells) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    cudaFree(dT);
    cudaFree(dF);
    heddle_place_destroy(x);
    return HEDDLE_E_NOMEM;
  }
  ok = cudaMemcpy(x->d_prof_deg, c->degrees, 4 * (size_t)x->D, cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(dT, c->T, es * (size_t)x->D, cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(dF, c->F, es * (size_t)x->D * c->s_max, cudaMemcpyHostToDevice) == cudaSuccess;
  if (ok) {
    dim3 grid((x->gstride + 255) / 256, x->D);
    if (c->dtype == HEDDLE_F32 || c->dtype == HEDDLE_F32X)
      k1_cost_tables<HEDDLE_F32><<<grid, 256>>>(dT, dF, x->D, c->s_max, x->gstride, x->d_gtab);
    else if (c->dtype == HEDDLE_F64) k1_cost_tables<HEDDLE_F64><<<grid, 256>>>(dT, dF, x->D, c->s_max, x->gstride, x->d_gtab);
    else k1_cost_tables<HEDDLE_U32><<<grid, 256>>>(dT, dF, x->D, c->s_max, x->gstride, x->d_gtab);
    x->launches++;
    ok = cudaGetLastError() == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess;
  }
  cudaFree(dT);
  cudaFree(dF);
  if (!ok) {
    heddle_place_destroy(x);
    return HEDDLE_E_CUDA;
  }
  // opt in to large dynamic shared memory for every K2 variant this ctx may launch
  // (the dynamic limit is the opt-in maximum minus the kernel's static shared memory)
  for (int kp = 0; kp < 2; ++kp)
    for (int kv = 0; kv < 4; ++kv) {
      const void* fn = reinterpret_cast<const void*>(k2_for(x->dtype, x->semiring, kp, kv & 1, kv >> 1));
      cudaFuncAttributes fa{};
      if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess ||
          cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               x->smem_optin - (int)fa.sharedSizeBytes) != cudaSuccess) {
        heddle_place_destroy(x);
        return HEDDLE_E_CUDA;
      }
      x->k2_smem_max = x->smem_optin - (int)fa.sharedSizeBytes;
    }
  if (c->flags & HEDDLE_VALLEY) {
    x->k8_smem_max = x->smem_optin;
    for (int v = 0; v < 24; ++v) {
      const void* fn = reinterpret_cast<const void*>(k8_for(x->dtype, v & 1, (v >> 1) & 1, (v >> 2) & 1, v >> 3));
      cudaFuncAttributes fa{};
      if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess ||
          cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               x->smem_optin - (int)fa.sharedSizeBytes) != cudaSuccess) {
        heddle_place_destroy(x);
        return HEDDLE_E_CUDA;
      }
      x->k8_smem_max = std::min(x->k8_smem_max, x->smem_optin - (int)fa.sharedSizeBytes);
    }
    for (int v = 0; v < 12; ++v) {
      const void* fn = reinterpret_cast<const void*>(k8c_for(x->dtype, v & 1, (v >> 1) & 1, v >> 2));
      cudaFuncAttributes fa{};
      if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess ||
          cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               x->smem_optin - (int)fa.sharedSizeBytes) != cudaSuccess) {
        heddle_place_destroy(x);
        return HEDDLE_E_CUDA;
      }
      x->k8_smem_max = std::min(x->k8_smem_max, x->smem_optin - (int)fa.sharedSizeBytes);
    }
  }
  *out = x;
  return HEDDLE_OK;
}

// K8L path (valley solver, n too large for shared memory): [fill parents] + prologue (validation,
// prefix sums, layer 1) + one launch per layer + finaliser.
heddle_status solve_valley_layered(heddle_place_ctx* x, SolveArgs& a, bool kp, bool kv, cudaStream_t s) {
  const int dt = x->dtype, sr = x->semiring;
  const int n = a.n, m = a.m, B = a.B;
  if (kp) {   // parents off the computed region read -1
    const int64_t cells = (int64_t)B * (m + 1) * (n + 1);
    const int fill_grid = (int)std::min<int64_t>((cells + 255) / 256, (int64_t)x->num_sms * 16);
    HP_DISPATCH(fill_launch, a, cells, fill_grid, s);
    x->launches++;
  }
  if (!x->vws.mask) {   // range-minimum workspace, sized for the context's limits
    const int nbm = vblocks(x->max_n), lvm = vlevels(nbm);
    const size_t des = dp_elem_size(x->dtype, x->semiring);
    void* mk = nullptr;
    void *bm = nullptr, *sp = nullptr, *smd = nullptr, *dl = nullptr, *dr = nullptr, *dn = nullptr, *kh = nullptr;
    if (cudaMalloc(&mk, 4 * 2 * (size_t)x->max_batch * nbm * kVBlk) != cudaSuccess ||
        cudaMalloc(&bm, des * 2 * (size_t)x->max_batch * nbm) != cudaSuccess ||
        cudaMalloc(&sp, des * (size_t)x->max_batch * std::max(1, lvm - 1) * nbm) != cudaSuccess ||
        cudaMalloc(&smd, des * (size_t)x->max_batch * (x->max_n + 1)) != cudaSuccess ||
        cudaMalloc(&dl, 4 * (size_t)x->max_batch) != cudaSuccess ||
        cudaMalloc(&dr, 4 * 2 * (size_t)x->max_batch) != cudaSuccess ||
        cudaMalloc(&dn, 4 * (size_t)x->max_batch) != cudaSuccess ||
        cudaMalloc(&kh, 4 * 2 * (size_t)x->max_batch * (x->max_n + 1)) != cudaSuccess ||
        cudaMemsetAsync(kh, 0xFF, 4 * 2 * (size_t)x->max_batch * (x->max_n + 1), s) != cudaSuccess) {
      cudaGetLastError();
      for (void* q : {mk, bm, sp, smd, dl, dr, dn, kh}) cudaFree(q);
      return HEDDLE_E_NOMEM;
    }
    x->vws = ValleyWs{static_cast<uint32_t*>(mk), bm, sp, smd, static_cast<int*>(dl), static_cast<int*>(dr),
                      static_cast<unsigned*>(dn), static_cast<int*>(kh), nbm, lvm, x->max_n};
  }
  // per solve: no in-run descents yet, no finished CTAs (the last CTA of each layer resets both)
  if (cudaMemsetAsync(x->vws.dlrun, 0xFF, 4 * 2 * (size_t)B, s) != cudaSuccess ||
      cudaMemsetAsync(x->vws.done, 0, 4 * (size_t)B, s) != cudaSuccess)
    return HEDDLE_E_CUDA;
  if (!x->d_rowcap) {
    if (cudaMalloc(&x->d_rowcap, sizeof(int2) * (size_t)x->max_batch * x->max_m) != cudaSuccess) { cudaGetLastError(); return HEDDLE_E_NOMEM; }
  }
  a.rowcap = x->d_rowcap;   // {profile row, cap} per worker: one load per layer launch
  pro_for(dt, sr, kp, kv)<<<B, kProThreads, 0, s>>>(a);   // (also the weight prefix sums, R5)
  x->launches++;
  K8LFn fn = k8l_for(dt, kp, kv, a.w != nullptr);
  // programmatic dependent launch: layer j+1's CTAs are scheduled while layer j runs and wait in
  // griddepcontrol.wait for its completion (no launch gap on the layer chain)
  static const bool pdl = !std::getenv("HEDDLE_PLACE_NO_PDL");   // A/B switch
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr.val.programmaticStreamSerializationAllowed = 1;
  for (int j = 1; j <= m; ++j) {
    const int ilo = (j == 1) ? 1 : (j == m ? n : j), ihi = (j == 1 || j < m) ? n - m + j : n;
    const int warps = ((ihi >> 5) - (ilo >> 5) + kK8LRun) / kK8LRun;
    // (row j's range-minimum extras are built by the last CTA of the launch to finish)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((warps + kK8LWarps - 1) / kK8LWarps, B);
    cfg.blockDim = dim3(32 * kK8LWarps);
    cfg.stream = s;
    cfg.attrs = &attr;
    cfg.numAttrs = pdl ? 1 : 0;
    if (cudaLaunchKernelEx(&cfg, fn, a, j, x->vws) != cudaSuccess) return HEDDLE_E_CUDA;
    x->launches++;
  }
  HP_DISPATCH(finalize_launch, a, s);
  x->launches++;
  return cudaGetLastError() == cudaSuccess ? HEDDLE_OK : HEDDLE_E_CUDA;
}

static heddle_status solve_impl(heddle_place_ctx* x, const heddle_place_problem* p, void* objective_out,
                                int32_t* status_out, void* stream, const unsigned* ready, unsigned ready_epoch,
                                int ready_chunk);

heddle_status heddle_place_solve(heddle_place_ctx* x, const heddle_place_problem* p, void* objective_out,
                                 int32_t* status_out, void* stream) {
  return solve_impl(x, p, objective_out, status_out, stream, nullptr, 0, 1);
}

static heddle_status solve_impl(heddle_place_ctx* x, const heddle_place_problem* p, void* objective_out,
                                int32_t* status_out, void* stream, const unsigned* ready, unsigned ready_epoch,
                                int ready_chunk) {
  if (!x || !p || !objective_out || !p->lengths || !p->degrees) return HEDDLE_E_INVALID;
  if (p->n < 1 || p->m < 1 || p->B < 1 || p->n > x->max_n || p->m > x->max_m || p->B > x->max_batch)
    return HEDDLE_E_INVALID;
  if (p->lengths_stride < 0 || p->degrees_stride < 0 || p->caps_stride < 0 || p->kv_caps_stride < 0)
    return HEDDLE_E_INVALID;
  const bool kv = p->kv_caps != nullptr;
  const bool kp = (x->flags & HEDDLE_KEEP_PARENTS) != 0;
  const bool wt = p->weights != nullptr;
  if (wt && p->weights_stride < 0) return HEDDLE_E_INVALID;
  const bool valley = (x->flags & HEDDLE_VALLEY) != 0;
  const int smem2 = valley ? k8_smem(x->dtype, p->n, p->m, kv, wt) : k2_smem(x->dtype, x->semiring, p->n, p->m, kv, wt);
  const bool fits = smem2 <= (valley ? x->k8_smem_max : x->k2_smem_max);
  const bool wide = dp_elem_size(x->dtype, x->semiring) == 8;
  const bool ragged = p->ms != nullptr || p->ns != nullptr;   // per-problem sizes: one-CTA-per-problem kernels only
  const bool layered = !ragged && !per_problem_kernel(x, p->n, p->m, p->B, kv, wt);
  if (!layered && !fits) return HEDDLE_E_INVALID;   // n too large for the one-CTA-per-problem kernel
  if (layered && kp && wide && !valley) return HEDDLE_E_INVALID;   // packed (value, split) atomics: 32-bit values
  if (x->split_world > 1 && (!layered || kp || wt)) return HEDDLE_E_INVALID;  // split mode: layered, no parent table, no weights
  DeviceGuard guard(x->device);
  SolveArgs a{};
  a.n = p->n;
  a.m = p->m;
  a.B = p->B;
  a.lengths = p->lengths;
  a.ls = p->lengths_stride;
  a.degrees = p->degrees;
  a.ds = p->degrees_stride;
  a.caps = p->caps;
  a.cs = p->caps_stride;
  a.kv = p->kv_caps;
  a.kvs = p->kv_caps_stride;
  a.w = p->weights;
  a.ws = p->weights_stride;
  a.ms = p->ms;
  a.ns = p->ns;
  if (wt && !x->d_wp) {
    if (cudaMalloc(&x->d_wp, 4 * (size_t)x->max_batch * (x->max_n + 1)) != cudaSuccess) { cudaGetLastError(); return HEDDLE_E_NOMEM; }
  }
  a.wpws = x->d_wp;
  a.gtab = x->d_gtab;
  a.gstride = x->gstride;
  a.prof_deg = x->d_prof_deg;
  a.D = x->D;
  a.lmax_u32 = x->lmax_u32;
  a.dpws = x->d_dp;
  a.parws = x->d_par;
  a.spws = x->d_sp;
  a.status = x->d_status;
  a.status_out = status_out;
  a.objective = objective_out;
  a.vscan = kScanPrefix;
  if (const char* e = std::getenv("HEDDLE_PLACE_VALLEY_SCAN")) a.vscan = std::atoi(e);   // tests / tuning
  a.ready = layered ? nullptr : ready;   // the pipelined inputs are only ever gated for the batched kernel
  a.ready_epoch = ready_epoch;
  a.ready_chunk = ready_chunk;
  if (layered && ready) return HEDDLE_E_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (valley) {
    const heddle_status st = layered ? solve_valley_layered(x, a, kp, kv, s) : HEDDLE_OK;
    if (st != HEDDLE_OK) return st;
    if (!layered) {
      // 1024-thread CTAs when problems are fewer than SMs (measured: 128-thread CTAs take the
      // rollout solve from 104 to 148 us, the TP sweep from 0.37 to 1.29 ms)
      int wide_min_n = 0;
      if (const char* e = std::getenv("HEDDLE_PLACE_K8_WIDE_MIN_N")) wide_min_n = std::atoi(e);   // tuning
      const bool wide_cta = p->B < x->num_sms && p->n >= wide_min_n;
      // at most 512 states per layer: 512 threads (one state each, as with 1024, without the idle
      // warps' instructions)
      int mid_max_n = 512 + 64;
      if (const char* e = std::getenv("HEDDLE_PLACE_K8_MID_MAX_N")) mid_max_n = std::atoi(e);   // tuning
      const int variant = wide_cta ? (p->n - p->m + 1 <= 512 && p->n <= mid_max_n ? 2 : 1) : 0;
      const int nthreads = variant == 2 ? kK8ThreadsMid : variant == 1 ? kK8ThreadsWide : kK8Threads;
      // few small problems: keep every dp row in shared memory and backtrack inside the kernel
      // (the latency of the rollout-sized call; heddle_place_backtrack then only copies)
      const size_t tab = dp_elem_size(x->dtype, x->semiring) * (size_t)(p->m + 1) * (p->n + 1);
      const bool fused = p->B < x->num_sms && !kp && (size_t)smem2 + tab <= (size_t)x->k8_smem_max;
      int smem_launch = smem2;
      if (fused) {
        if (!x->d_fbounds && cudaMalloc(&x->d_fbounds, 4 * (size_t)x->max_batch * (x->max_m + 1)) != cudaSuccess) {
          cudaGetLastError();
          return HEDDLE_E_NOMEM;
        }
        if (cudaMemsetAsync(x->d_fbounds, 0xFF, 4 * (size_t)p->B * (p->m + 1), s) != cudaSuccess) return HEDDLE_E_CUDA;
        a.fbounds = x->d_fbounds;
        smem_launch = smem2 + (int)tab;
      }
      // a few problems: a cluster of kK8Cluster CTAs per problem (each computes a quarter of every
      // layer's states into every CTA's copy of the row over distributed shared memory)
      const char* cle = std::getenv("HEDDLE_PLACE_K8_CLUSTER");   // 0 off, 1 auto (default), 2 always (tests)
      const int cl_mode = cle ? std::atoi(cle) : 1;
      const int states = p->n - p->m + 1;
      int cv = 0;   // 512 threads x 8 CTAs (measured best on the TP sweep and the §6.2 size)
      if (const char* e = std::getenv("HEDDLE_PLACE_K8_CLUSTER_V")) cv = std::atoi(e);   // tuning
      const int csize = cv == 0 ? 2 * kK8Cluster : kK8Cluster;
      // (rollout-sized layers stay on one CTA: the cluster barrier costs more than it saves there)
      const bool cluster = cl_mode != 0 && wide_cta && !kp && (states > 640 || cl_mode == 2) &&
                           (int64_t)p->B * csize <= x->num_sms;
      if (cluster) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(p->B * csize);
        cfg.blockDim = dim3(cv == 2 ? 1024 : 512);
        cfg.dynamicSmemBytes = smem_launch;
        cfg.stream = s;
        cudaLaunchAttribute attr{};
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = csize;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, k8c_for(x->dtype, kv, wt, cv), a) != cudaSuccess) return HEDDLE_E_CUDA;
      } else {
        k8_for(x->dtype, kp, kv, wt, variant)<<<p->B, nthreads, smem_launch, s>>>(a);
      }
      x->launches++;
      if (cudaGetLastError() != cudaSuccess) return HEDDLE_E_CUDA;
    }
  } else if (!layered) {
    k2_for(x->dtype, x->semiring, kp, kv, wt)<<<p->B, kK2Threads, smem2, s>>>(a);
    x->launches++;
    if (cudaGetLastError() != cudaSuccess) return HEDDLE_E_CUDA;
  } else {
    const heddle_status st = solve_layered(x, a, kp, kv, s);
    if (st != HEDDLE_OK) return st;
  }
  x->last = a;
  x->last_fused = a.fbounds != nullptr;
  x->last_kv = kv;
  x->last_w = wt;
  x->last_layered = layered;
  x->solved = true;
  return HEDDLE_OK;
}

heddle_status heddle_place_backtrack(heddle_place_ctx* x, int32_t* boundaries_out, int32_t* parents_out,
                                     void* stream) {
  if (!x || !boundaries_out) return HEDDLE_E_INVALID;
  if (!x->solved) return HEDDLE_E_STATE;
  if (parents_out && !(x->flags & HEDDLE_KEEP_PARENTS)) return HEDDLE_E_STATE;
  if (parents_out && x->last.ns) return HEDDLE_E_INVALID;   // ragged n: rows are packed per problem
  DeviceGuard guard(x->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const SolveArgs& a = x->last;
  if (x->last_fused && !parents_out)   // the valley kernel already walked the back-pointers
    return cudaMemcpyAsync(boundaries_out, x->d_fbounds, 4 * (size_t)a.B * (a.m + 1), cudaMemcpyDeviceToDevice, s) ==
                   cudaSuccess ? HEDDLE_OK : HEDDLE_E_CUDA;
  // few min-plus problems: a CTA per problem (the cost bound prunes little there, so the
  // lowest-argmin scan can cover tens of thousands of splits per layer at large n)
  if (a.B < x->num_sms && x->semiring == HEDDLE_MINPLUS)
    k4c_for(x->dtype, x->semiring, x->last_kv, x->last_w)<<<a.B, kK4CtaThreads, 0, s>>>(a, boundaries_out);
  else
    k4_for(x->dtype, x->semiring, x->last_kv, x->last_w)<<<(a.B + kK4Warps - 1) / kK4Warps, 32 * kK4Warps, 0, s>>>(
        a, boundaries_out);
  x->launches++;
  if (cudaGetLastError() != cudaSuccess) return HEDDLE_E_CUDA;
  if (parents_out) {
    const size_t row = 4 * (size_t)(a.n + 1);
    if (cudaMemcpy2DAsync(parents_out, row * a.m, x->d_par + (size_t)(a.n + 1), row * (a.m + 1), row * a.m, a.B,
                          cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return HEDDLE_E_CUDA;
  }
  return HEDDLE_OK;
}

heddle_status heddle_place_query(heddle_place_ctx* x, int32_t nq, const int32_t* qb, const int32_t* qj,
                                 const int32_t* qi, void* dp_out, int32_t* parents_out, void* stream) {
  if (!x || nq < 0 || (nq > 0 && (!qb || !qj || !qi || !dp_out || !parents_out))) return HEDDLE_E_INVALID;
  if (!x->solved) return HEDDLE_E_STATE;
  if (nq == 0) return HEDDLE_OK;
  DeviceGuard guard(x->device);
  const SolveArgs& a = x->last;
  const int dt = x->dtype, sr = x->semiring;
  (void)dt; (void)sr;
  k4q_for(x->dtype, x->semiring, x->last_kv, x->last_w)<<<(nq + kK4Warps - 1) / kK4Warps, 32 * kK4Warps, 0,
                                                          static_cast<cudaStream_t>(stream)>>>(a, nq, qb, qj, qi,
                                                                                               dp_out, parents_out);
  x->launches++;
  return cudaGetLastError() == cudaSuccess ? HEDDLE_OK : HEDDLE_E_CUDA;
}

heddle_status heddle_place_solve_host(heddle_place_ctx* x, const heddle_place_problem* hp_, void* objective_host,
                                      int32_t* boundaries_host, int32_t* status_host, void* stream,
                                      int64_t* bytes_h2d, int64_t* bytes_d2h) {
  if (!x || !hp_ || !objective_host || !boundaries_host || !hp_->lengths || !hp_->degrees) return HEDDLE_E_INVALID;
  const heddle_place_problem& p = *hp_;
  if (p.n < 1 || p.m < 1 || p.B < 1 || p.n > x->max_n || p.m > x->max_m || p.B > x->max_batch)
    return HEDDLE_E_INVALID;
  DeviceGuard guard(x->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t es = elem_size(x->dtype);
  const size_t oes = dp_elem_size(x->dtype, x->semiring);
  const int64_t B = p.B, n = p.n, m = p.m;
  const int64_t lrows = p.lengths_stride == 0 ? 1 : B;
  const int64_t drows = p.degrees_stride == 0 ? 1 : B;
  const int64_t crows = p.caps ? (p.caps_stride == 0 ? 1 : B) : 0;
  const int64_t krows = p.kv_caps ? (p.kv_caps_stride == 0 ? 1 : B) : 0;
  const int64_t wrows = p.weights ? (p.weights_stride == 0 ? 1 : B) : 0;
  auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
  const size_t bl = al(es * lrows * n), bd = al(4 * drows * m), bc = al(4 * crows * m), bk = al(8 * krows * m);
  const size_t bw = al(4 * wrows * n), bm = p.ms ? al(4 * B) : 0, bn = p.ns ? al(4 * B) : 0;
  const size_t bo = al(8 * B), bb = al(4 * B * (m + 1)), bs = al(4 * B);
  const size_t need = bl + bd + bc + bk + bo + bb + bs + bw + bm + bn;
  if (need > x->stage_bytes) {
    cudaFree(x->d_stage);
    x->d_stage = nullptr;
    x->stage_bytes = 0;
    if (cudaMalloc(&x->d_stage, need) != cudaSuccess) { cudaGetLastError(); return HEDDLE_E_NOMEM; }
    x->stage_bytes = need;
  }
  char* base = static_cast<char*>(x->d_stage);
  char *dl = base, *dd = dl + bl, *dc = dd + bd, *dk = dc + bc, *dob = dk + bk, *dbd = dob + bo, *dst = dbd + bb;
  char* dw = dst + bs;
  char* dms = dw + bw;
  char* dns = dms + bm;
  int64_t h2d = 0, d2h = 0;
  // Pipelined inputs (batched kernel, many problems): the host->device copies run on a copy stream
  // in chunks of problems, each chunk followed by a 4-byte copy of the call's epoch into its ready
  // flag; the ONE K2 launch on the caller's stream starts at once and each CTA waits (thread 0,
  // acquire poll) for its problem's chunk, so only the first chunk's copy is exposed.  Copies run on
  // the copy engines, never on the SMs the waiting CTAs hold, so the wait always ends.
  const bool kv = p.kv_caps != nullptr, wt = p.weights != nullptr;
  const bool batched_path = p.ms != nullptr || p.ns != nullptr || per_problem_kernel(x, p.n, p.m, p.B, kv, wt);
  int64_t chunk = std::max<int64_t>(kPipeMinChunk, (B + kPipeChunks - 1) / kPipeChunks);
  if (const char* e = std::getenv("HEDDLE_PLACE_HOST_CHUNK")) chunk = std::max(1, std::atoi(e));   // tuning
  const int64_t chunks = batched_path ? (B + chunk - 1) / chunk : 1;
  const bool pipe = chunks > 1;
  if (pipe && !x->copy_stream) {
    bool ok = cudaStreamCreateWithFlags(&x->copy_stream, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&x->copy_done, cudaEventDisableTiming) == cudaSuccess &&
              cudaMalloc(&x->d_chunk_ready, 4 * (size_t)kPipeChunks * 2) == cudaSuccess &&
              cudaMemset(x->d_chunk_ready, 0, 4 * (size_t)kPipeChunks * 2) == cudaSuccess &&
              cudaHostAlloc(&x->h_epoch, 4, cudaHostAllocDefault) == cudaSuccess;
    if (!ok) { cudaGetLastError(); return HEDDLE_E_CUDA; }
  }
  if (pipe && chunks > 2 * kPipeChunks) return HEDDLE_E_INVALID;   // only reachable through the tuning knob
  cudaStream_t cs = pipe ? x->copy_stream : s;
  unsigned epoch = 0;
  if (pipe) {
    epoch = ++x->pipe_epoch;
    if (epoch == 0) epoch = ++x->pipe_epoch;     // 0 is the flags' initial value
    *x->h_epoch = epoch;                    // previous calls synchronised: no copy still reads it
  }
  auto up = [&](char* dbase, const void* src, int64_t rows, int64_t cols, int64_t stride, size_t esz, int64_t r0,
                int64_t r1) -> bool {
    if (rows == 0) return true;
    if (rows == 1) {   // broadcast row: copied once, with the first chunk
      if (r0 != 0) return true;
      r1 = 1;
    }
    const size_t w = esz * cols;
    h2d += (int64_t)(w * (r1 - r0));
    const char* hs = static_cast<const char*>(src) + esz * stride * r0;
    char* dd = dbase + w * r0;
    if (stride == cols || r1 - r0 == 1)
      return cudaMemcpyAsync(dd, hs, w * (r1 - r0), cudaMemcpyHostToDevice, cs) == cudaSuccess;
    return cudaMemcpy2DAsync(dd, w, hs, esz * stride, w, r1 - r0, cudaMemcpyHostToDevice, cs) == cudaSuccess;
  };
  if (pipe) {   // the copy stream must not overwrite staging a previous use of stream s still reads
    if (cudaEventRecord(x->copy_done, s) != cudaSuccess || cudaStreamWaitEvent(cs, x->copy_done, 0) != cudaSuccess)
      return HEDDLE_E_CUDA;
  }
  for (int64_t c = 0; c < chunks; ++c) {
    const int64_t b0 = c * chunk, b1 = pipe ? std::min(B, b0 + chunk) : B;
    if (!up(dl, p.lengths, lrows, n, p.lengths_stride, es, b0, b1) ||
        !up(dd, p.degrees, drows, m, p.degrees_stride, 4, b0, b1) ||
        !up(dc, p.caps, crows, m, p.caps_stride, 4, b0, b1) ||
        !up(dk, p.kv_caps, krows, m, p.kv_caps_stride, 8, b0, b1) ||
        !up(dw, p.weights, wrows, n, p.weights_stride, 4, b0, b1) ||
        !up(dms, p.ms, p.ms ? B : 0, 1, 1, 4, b0, b1) ||
        !up(dns, p.ns, p.ns ? B : 0, 1, 1, 4, b0, b1))
      return HEDDLE_E_CUDA;
    if (pipe && cudaMemcpyAsync(x->d_chunk_ready + c, x->h_epoch, 4, cudaMemcpyHostToDevice, cs) != cudaSuccess)
      return HEDDLE_E_CUDA;
  }
  if (pipe && cudaEventRecord(x->copy_done, cs) != cudaSuccess) return HEDDLE_E_CUDA;
  heddle_place_problem q = p;
  q.lengths = dl;
  q.lengths_stride = p.lengths_stride == 0 ? 0 : n;
  q.degrees = reinterpret_cast<const int32_t*>(dd);
  q.degrees_stride = p.degrees_stride == 0 ? 0 : m;
  q.caps = p.caps ? reinterpret_cast<const int32_t*>(dc) : nullptr;
  q.caps_stride = p.caps_stride == 0 ? 0 : m;
  q.kv_caps = p.kv_caps ? reinterpret_cast<const int64_t*>(dk) : nullptr;
  q.kv_caps_stride = p.kv_caps_stride == 0 ? 0 : m;
  q.weights = p.weights ? reinterpret_cast<const int32_t*>(dw) : nullptr;
  q.weights_stride = p.weights_stride == 0 ? 0 : n;
  q.ms = p.ms ? reinterpret_cast<const int32_t*>(dms) : nullptr;
  q.ns = p.ns ? reinterpret_cast<const int32_t*>(dns) : nullptr;
  heddle_status st =
      solve_impl(x, &q, dob, reinterpret_cast<int32_t*>(dst), stream, pipe ? x->d_chunk_ready : nullptr, epoch, (int)chunk);
  if (st != HEDDLE_OK) {
    if (pipe) cudaStreamSynchronize(cs);
    return st;
  }
  // stream order for everything after the kernel (the backtrack re-reads lengths; the next call's copies)
  if (pipe && cudaStreamWaitEvent(s, x->copy_done, 0) != cudaSuccess) return HEDDLE_E_CUDA;
  st = heddle_place_backtrack(x, reinterpret_cast<int32_t*>(dbd), nullptr, stream);
  if (st != HEDDLE_OK) return st;
  bool ok = cudaMemcpyAsync(objective_host, dob, oes * B, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
            cudaMemcpyAsync(boundaries_host, dbd, 4 * B * (m + 1), cudaMemcpyDeviceToHost, s) == cudaSuccess;
  d2h += (int64_t)(oes * B + 4 * B * (m + 1));
  if (ok && status_host) {
    ok = cudaMemcpyAsync(status_host, dst, 4 * B, cudaMemcpyDeviceToHost, s) == cudaSuccess;
    d2h += 4 * B;
  }
  if (!ok || cudaStreamSynchronize(s) != cudaSuccess) return HEDDLE_E_CUDA;
  if (bytes_h2d) *bytes_h2d = h2d;
  if (bytes_d2h) *bytes_d2h = d2h;
  return HEDDLE_OK;
}


heddle_status heddle_place_nccl_unique_id(void* id_out, int32_t bytes) {
  if (!id_out || bytes < (int32_t)sizeof(ncclUniqueId)) return HEDDLE_E_INVALID;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return HEDDLE_E_NCCL;
  std::memcpy(id_out, &id, sizeof(id));
  return HEDDLE_OK;
}

// Exchange CUDA IPC handles of the dp workspace and the arrival counters over NCCL and map
// every peer's buffers (NVLink peer memory).  Returns OK without enabling P2P when the
// devices cannot access each other (the NCCL all-gather exchange is used then).
static heddle_status setup_p2p(heddle_place_ctx* x) {
  const int world = x->split_world, rank = x->split_rank;
  DeviceGuard guard(x->device);
  const int ncb_max = (x->max_n + 3) / kK3Cols + 2;
  if (cudaMalloc(&x->d_flags, 8 * (size_t)(x->max_m + 2)) != cudaSuccess ||   // [max_m+1]: K5 arrivals
      cudaMemset(x->d_flags, 0, 8 * (size_t)(x->max_m + 2)) != cudaSuccess ||
      cudaMalloc(&x->d_peer_arrive, sizeof(void*) * world) != cudaSuccess ||
      cudaMalloc(&x->d_blkdone, sizeof(unsigned) * (size_t)x->max_batch * ncb_max * (x->max_m + 1)) != cudaSuccess ||
      cudaMalloc(&x->d_err, sizeof(int)) != cudaSuccess || cudaMemset(x->d_err, 0, sizeof(int)) != cudaSuccess ||
      cudaMalloc(&x->d_peer_dp, sizeof(void*) * world) != cudaSuccess ||
      cudaMalloc(&x->d_peer_flags, sizeof(void*) * world) != cudaSuccess ||
      cudaMalloc(&x->d_peer_ready, sizeof(void*) * world) != cudaSuccess ||
      (!x->d_ready && (cudaMalloc(&x->d_ready, 8 * (size_t)(x->max_m + 1) * x->max_batch * ncb_max) != cudaSuccess ||
                       cudaMemset(x->d_ready, 0, 8 * (size_t)(x->max_m + 1) * x->max_batch * ncb_max) != cudaSuccess))) {
    cudaGetLastError();
    return HEDDLE_E_NOMEM;
  }
  cudaIpcMemHandle_t mine[3];
  if (cudaIpcGetMemHandle(&mine[0], x->d_dp) != cudaSuccess || cudaIpcGetMemHandle(&mine[1], x->d_flags) != cudaSuccess ||
      cudaIpcGetMemHandle(&mine[2], x->d_ready) != cudaSuccess) {
    cudaGetLastError();
    return HEDDLE_OK;   // no IPC: keep the NCCL exchange
  }
  char *dsend = nullptr, *drecv = nullptr;
  const size_t hb = sizeof(mine);
  if (cudaMalloc(&dsend, hb) != cudaSuccess || cudaMalloc(&drecv, hb * world) != cudaSuccess) return HEDDLE_E_NOMEM;
  cudaMemcpy(dsend, mine, hb, cudaMemcpyHostToDevice);
  ncclResult_t nr = ncclAllGather(dsend, drecv, hb, ncclChar, x->comm, 0);
  std::vector<cudaIpcMemHandle_t> all(3 * world);
  if (nr == ncclSuccess) cudaMemcpy(all.data(), drecv, hb * world, cudaMemcpyDeviceToHost);
  cudaFree(dsend);
  cudaFree(drecv);
  if (nr != ncclSuccess) return HEDDLE_E_NCCL;
  // every rank must be able to reach every peer; decide collectively (min over ranks)
  int ok = 1;
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  x->peer_dp_h.assign(world, nullptr);
  x->peer_flags_h.assign(world, nullptr);
  x->peer_ready_h.assign(world, nullptr);
  for (int r = 0; r < world && ok; ++r) {
    if (r == rank) {
      x->peer_dp_h[r] = x->d_dp;
      x->peer_flags_h[r] = x->d_flags;
      x->peer_ready_h[r] = x->d_ready;
      continue;
    }
    if (cudaIpcOpenMemHandle(&x->peer_dp_h[r], all[3 * r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&x->peer_flags_h[r], all[3 * r + 1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&x->peer_ready_h[r], all[3 * r + 2], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
    }
  }
  int* dok = nullptr;
  cudaMalloc(&dok, sizeof(int));
  cudaMemcpy(dok, &ok, sizeof(int), cudaMemcpyHostToDevice);
  nr = ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, x->comm, 0);
  cudaMemcpy(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(dok);
  if (nr != ncclSuccess) return HEDDLE_E_NCCL;
  if (!ok) {
    for (int r = 0; r < world; ++r) {
      if (r == rank) continue;
      if (x->peer_dp_h[r]) cudaIpcCloseMemHandle(x->peer_dp_h[r]);
      if (x->peer_flags_h[r]) cudaIpcCloseMemHandle(x->peer_flags_h[r]);
      if (x->peer_ready_h[r]) cudaIpcCloseMemHandle(x->peer_ready_h[r]);
    }
    x->peer_dp_h.clear();
    x->peer_flags_h.clear();
    x->peer_ready_h.clear();
    return HEDDLE_OK;
  }
  cudaMemcpy(x->d_peer_dp, x->peer_dp_h.data(), sizeof(void*) * world, cudaMemcpyHostToDevice);
  cudaMemcpy(x->d_peer_flags, x->peer_flags_h.data(), sizeof(void*) * world, cudaMemcpyHostToDevice);
  cudaMemcpy(x->d_peer_ready, x->peer_ready_h.data(), sizeof(void*) * world, cudaMemcpyHostToDevice);
  {
    std::vector<unsigned long long*> arr(world);
    for (int r = 0; r < world; ++r) arr[r] = static_cast<unsigned long long*>(x->peer_flags_h[r]) + x->max_m + 1;
    cudaMemcpy(x->d_peer_arrive, arr.data(), sizeof(void*) * world, cudaMemcpyHostToDevice);
  }
  x->p2p = cudaGetLastError() == cudaSuccess;
  return HEDDLE_OK;
}

heddle_status heddle_place_init_split(const heddle_place_config* cfg, const void* nccl_unique_id, int32_t rank,
                                      int32_t world, heddle_place_ctx** out) {
  if (!out) return HEDDLE_E_INVALID;
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world || (cfg && (cfg->flags & (HEDDLE_KEEP_PARENTS | HEDDLE_VALLEY))))
    return HEDDLE_E_INVALID;
  if (nccl_unique_id == nullptr && rank != 0) return HEDDLE_E_INVALID;   // emulation: one process
  heddle_place_config c = *cfg;
  c.flags |= HEDDLE_FORCE_LAYERED;
  heddle_place_ctx* x = nullptr;
  heddle_status st = heddle_place_init(&c, &x);
  if (st != HEDDLE_OK) return st;
  x->split_world = world;
  x->split_rank = rank;
  if (world > 1) {
    if (nccl_unique_id == nullptr) {
      x->split_emulate = true;
    } else {
      DeviceGuard guard(x->device);
      ncclUniqueId id;
      std::memcpy(&id, nccl_unique_id, sizeof(id));
      if (ncclCommInitRank(&x->comm, world, id, rank) != ncclSuccess) {
        x->comm = nullptr;
        heddle_place_destroy(x);
        return HEDDLE_E_NCCL;
      }
      const char* ex = std::getenv("HEDDLE_PLACE_EXCHANGE");   // "nccl" forces the all-gather exchange
      if (!(ex && std::strcmp(ex, "nccl") == 0)) {
        st = setup_p2p(x);
        if (st != HEDDLE_OK) {
          heddle_place_destroy(x);
          return st;
        }
      }
    }
  }
  *out = x;
  return HEDDLE_OK;
}

int32_t heddle_place_split_plan(int32_t n, int32_t m, int32_t world, int32_t rank, int64_t* publishes_out,
                                int64_t* arrivals_out) {
  if (n < 1 || m < 1 || n < m || world < 1 || rank < 0 || rank >= world || !publishes_out || !arrivals_out)
    return -1;
  split_traffic(n, m, world, rank, publishes_out, arrivals_out);
  return 0;
}

int32_t heddle_place_split_blocks(int32_t ncb, int32_t world, int32_t rank, int32_t* blocks_out, int32_t cap) {
  if (ncb < 0 || world < 1 || rank < 0 || rank >= world) return -1;
  const int slots = owned_slots(ncb, world);
  int cnt = 0;
  for (int sl = 0; sl < slots; ++sl) {
    const int b = owned_block(sl, rank, world);
    if (b < ncb) {
      if (blocks_out && cnt < cap) blocks_out[cnt] = b;
      ++cnt;
    }
  }
  return cnt;
}


int64_t heddle_place_debug_violations(void) {
#ifdef HEDDLE_CHECK_BOUNDS
  unsigned long long v = 0;
  if (cudaMemcpyFromSymbol(&v, g_hp_violations, sizeof(v)) != cudaSuccess) return -2;
  return (int64_t)v;
#else
  return -1;
#endif
}


heddle_status heddle_place_retarget(const int32_t* boundaries, int32_t m, int32_t B, const int32_t* n_active,
                                    const int32_t* query_problem, const int32_t* query_rank, int32_t nq,
                                    int32_t* worker_out, void* stream) {
  if (!boundaries || !n_active || !query_problem || !query_rank || !worker_out || m < 1 || B < 1 || nq < 0)
    return HEDDLE_E_INVALID;
  if (nq == 0) return HEDDLE_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int grid = (int)std::min<int64_t>((nq + 255) / 256, 4096);
  k6_retarget<<<grid, 256, 0, s>>>(boundaries, m, B, n_active, query_problem, query_rank, nq, worker_out);
  return cudaGetLastError() == cudaSuccess ? HEDDLE_OK : HEDDLE_E_CUDA;
}


heddle_status heddle_place_objective(heddle_place_ctx* x, const heddle_place_problem* p, void* objective_out,
                                     int32_t* status_out, void* stream) {
  if (!x || !p || !objective_out || !p->lengths || !p->degrees) return HEDDLE_E_INVALID;
  if (p->n < 1 || p->m < 1 || p->B < 1 || p->n > x->max_n || p->m > x->max_m || p->B > x->max_batch)
    return HEDDLE_E_INVALID;
  if (x->semiring != HEDDLE_MINMAX || p->weights || x->split_world > 1) return HEDDLE_E_INVALID;
  if (p->lengths_stride < 0 || p->degrees_stride < 0 || p->caps_stride < 0 || p->kv_caps_stride < 0)
    return HEDDLE_E_INVALID;
  DeviceGuard guard(x->device);
  SolveArgs a{};
  a.n = p->n;
  a.m = p->m;
  a.B = p->B;
  a.lengths = p->lengths;
  a.ls = p->lengths_stride;
  a.degrees = p->degrees;
  a.ds = p->degrees_stride;
  a.caps = p->caps;
  a.cs = p->caps_stride;
  a.kv = p->kv_caps;
  a.kvs = p->kv_caps_stride;
  a.ms = p->ms;
  a.ns = p->ns;
  a.gtab = x->d_gtab;
  a.gstride = x->gstride;
  a.prof_deg = x->d_prof_deg;
  a.D = x->D;
  a.lmax_u32 = x->lmax_u32;
  a.spws = x->d_sp;
  a.status = x->d_status;
  a.status_out = status_out;
  a.objective = objective_out;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool kv = p->kv_caps != nullptr;
  const int grid = (p->B + kK7Warps - 1) / kK7Warps;
  // few problems: a CTA of 32 warps per problem (32-ary bisection); many: a warp per problem
  const bool wide = p->B < 4 * x->num_sms;
#define HP_K7(DT_)                                                                                 \
  do {                                                                                             \
    if (wide) {                                                                                    \
      if (kv) k7_parametric<DT_, true, 32><<<p->B, 1024, 0, s>>>(a);                              \
      else k7_parametric<DT_, false, 32><<<p->B, 1024, 0, s>>>(a);                                \
    } else {                                                                                       \
      if (kv) k7_parametric<DT_, true, 1><<<grid, 32 * kK7Warps, 0, s>>>(a);                      \
      else k7_parametric<DT_, false, 1><<<grid, 32 * kK7Warps, 0, s>>>(a);                        \
    }                                                                                              \
  } while (0)
  if (x->dtype == HEDDLE_F32) HP_K7(HEDDLE_F32);
  else if (x->dtype == HEDDLE_F64) HP_K7(HEDDLE_F64);
  else HP_K7(HEDDLE_U32);
#undef HP_K7
  x->launches++;
  x->solved = false;   // no dp rows: a following backtrack is a state error
  return cudaGetLastError() == cudaSuccess ? HEDDLE_OK : HEDDLE_E_CUDA;
}

heddle_status heddle_place_aggregate(int32_t dtype, const void* lengths, int64_t lengths_stride, int32_t n, int32_t B,
                                    double threshold, int32_t bucket, void* agg_lengths_out, int32_t* weights_out,
                                    int32_t* starts_out, int32_t* n_out, void* stream) {
  if (!lengths || !agg_lengths_out || !weights_out || !starts_out || !n_out || n < 1 || B < 1 || bucket < 1 ||
      lengths_stride < 0 || std::isnan(threshold))
    return HEDDLE_E_INVALID;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == HEDDLE_F32 || dtype == HEDDLE_F32X)
    k10_aggregate<float><<<B, 128, 0, s>>>(static_cast<const float*>(lengths), lengths_stride, n, threshold, bucket,
                                           static_cast<float*>(agg_lengths_out), weights_out, starts_out, n_out);
  else if (dtype == HEDDLE_F64)
    k10_aggregate<double><<<B, 128, 0, s>>>(static_cast<const double*>(lengths), lengths_stride, n, threshold, bucket,
                                            static_cast<double*>(agg_lengths_out), weights_out, starts_out, n_out);
  else if (dtype == HEDDLE_U32)
    k10_aggregate<uint32_t><<<B, 128, 0, s>>>(static_cast<const uint32_t*>(lengths), lengths_stride, n, threshold,
                                              bucket, static_cast<uint32_t*>(agg_lengths_out), weights_out,
                                              starts_out, n_out);
  else
    return HEDDLE_E_INVALID;
  return cudaGetLastError() == cudaSuccess ? HEDDLE_OK : HEDDLE_E_CUDA;
}

heddle_status heddle_place_expand(const int32_t* agg_boundaries, int32_t m, int32_t B, const int32_t* starts, int32_t n,
                                  int32_t* boundaries_out, void* stream) {
  if (!agg_boundaries || !starts || !boundaries_out || m < 1 || B < 1 || n < 1) return HEDDLE_E_INVALID;
  const int64_t total = (int64_t)B * (m + 1);
  k10_expand<<<(unsigned)((total + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(agg_boundaries, m, B,
                                                                                             starts, n, boundaries_out);
  return cudaGetLastError() == cudaSuccess ? HEDDLE_OK : HEDDLE_E_CUDA;
}

heddle_status heddle_place_anneal(heddle_place_ctx* x, const heddle_place_anneal_args* A, heddle_place_anneal_out* O,
                                  void* stream) {
  if (!x || !A || !O || !A->lengths || !A->init_degrees || !A->init_m || !A->uniforms || !O->best_makespan ||
      !O->best_degrees || !O->best_m)
    return HEDDLE_E_INVALID;
  const int P = A->chains, M = A->m_max, n = A->n;
  if (P < 1 || P > 1024 || P > x->max_batch || M < 1 || M > x->max_m || n < 1 || n > x->max_n || A->m_min < 1 ||
      A->m_min > M || A->iters < 0 || x->D > kK9MaxD || x->split_world > 1 || !(A->cooling > 0.0 && A->cooling < 1.0))
    return HEDDLE_E_INVALID;
  DeviceGuard guard(x->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // workspace: degree rows (cur, prop), counters, per-chain doubles, the solver's objective / status
  auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
  const size_t rows = al(4 * (size_t)P * M), ints = al(4 * (size_t)P), dbl = al(8 * (size_t)P);
  const size_t need = 2 * rows + 3 * ints + 3 * dbl + al(4) + al(8 * (size_t)P) + ints + al(4 * (size_t)x->D);
  if (need > x->sa_bytes) {
    cudaFree(x->d_sa);
    x->d_sa = nullptr;
    x->sa_bytes = 0;
    if (cudaMalloc(&x->d_sa, need) != cudaSuccess) { cudaGetLastError(); return HEDDLE_E_NOMEM; }
    x->sa_bytes = need;
  }
  if (!x->sa_stream && cudaStreamCreateWithFlags(&x->sa_stream, cudaStreamNonBlocking) != cudaSuccess)
    return HEDDLE_E_CUDA;
  char* w = static_cast<char*>(x->d_sa);
  AnnealArgs sa{};
  sa.P = P; sa.M = M; sa.n = n; sa.D = x->D;
  sa.m_min = A->m_min; sa.m_max = M;
  sa.u = A->uniforms; sa.iters = A->iters; sa.cooling = A->cooling;
  sa.cur_deg = reinterpret_cast<int*>(w); w += rows;
  sa.prop_deg = reinterpret_cast<int*>(w); w += rows;
  sa.cur_m = reinterpret_cast<int*>(w); w += ints;
  sa.prop_m = reinterpret_cast<int*>(w); w += ints;
  sa.live = reinterpret_cast<int*>(w); w += ints;
  sa.C = reinterpret_cast<double*>(w); w += dbl;
  sa.T = reinterpret_cast<double*>(w); w += dbl;
  sa.eps = reinterpret_cast<double*>(w); w += dbl;
  sa.it = reinterpret_cast<int*>(w); w += al(4);
  void* obj = w; w += al(8 * (size_t)P);
  int32_t* st = reinterpret_cast<int32_t*>(w); w += ints;
  int* deg_desc = reinterpret_cast<int*>(w);
  sa.deg_desc = deg_desc;
  sa.best = static_cast<double*>(O->best_makespan);
  sa.best_deg = O->best_degrees;
  sa.best_m = O->best_m;
  sa.trace_c = O->trace;
  sa.accepted = O->accepted;
  sa.obj = obj;
  sa.obj_kind = x->dtype == HEDDLE_F32 ? 0 : (x->dtype == HEDDLE_F64 || x->dtype == HEDDLE_F32X) ? 1
              : (x->semiring == HEDDLE_MINPLUS ? 3 : 2);
  std::vector<int> hdeg(x->prof_degrees);
  std::sort(hdeg.begin(), hdeg.end(), std::greater<int>());
  if (cudaMemcpyAsync(deg_desc, hdeg.data(), 4 * hdeg.size(), cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(sa.cur_deg, A->init_degrees, 4 * (size_t)P * M, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(sa.cur_m, A->init_m, 4 * (size_t)P, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return HEDDLE_E_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return HEDDLE_E_CUDA;   // hdeg is a host temporary
  // the PresortedDP makespans of one ragged batch of allocations (rows of `deg`, counts `ms`)
  auto evaluate = [&](const int* deg, const int* ms, cudaStream_t q) -> heddle_status {
    heddle_place_problem pb{};
    pb.n = n; pb.m = M; pb.B = P;
    pb.lengths = A->lengths; pb.lengths_stride = 0;
    pb.degrees = deg; pb.degrees_stride = M;
    pb.ms = ms;
    return A->objective_only ? heddle_place_objective(x, &pb, obj, st, q) : heddle_place_solve(x, &pb, obj, st, q);
  };
  // lines 1-4: the start states' makespans, T0, eps, best
  heddle_status e = evaluate(sa.cur_deg, sa.cur_m, s);
  if (e != HEDDLE_OK) return e;
  k9_start<<<(P + 127) / 128, 128, 0, s>>>(sa, A->eps_frac);
  x->launches++;
  // iteration count: every chain cools from its own T0 by the same factor and stops at
  // eps_frac * T0; replay the host arithmetic of the walk to find the last live iteration
  std::vector<double> hC(P);
  if (cudaMemcpyAsync(hC.data(), sa.C, 8 * (size_t)P, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return HEDDLE_E_CUDA;
  int nit = 0;
  for (int c = 0; c < P; ++c) {
    double T = hC[c];
    const double eps = A->eps_frac * hC[c];
    int k = 0;
    while (T > eps && k < A->iters) { T *= A->cooling; ++k; }
    nit = std::max(nit, k);
  }
  // lines 5-16: perturb -> ragged solve -> accept, captured once as a CUDA graph and replayed
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  bool graphed = false;
  if (nit > 1) {
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) {
      cudaEventRecord(ev, s);
      cudaStreamWaitEvent(x->sa_stream, ev, 0);
      cudaEventDestroy(ev);
    }
    const int64_t l0 = x->launches;
    if (cudaStreamBeginCapture(x->sa_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
      k9_perturb<<<(P + 127) / 128, 128, 0, x->sa_stream>>>(sa);
      const heddle_status ge = evaluate(sa.prop_deg, sa.prop_m, x->sa_stream);
      k9_accept<<<1, ((P + 31) / 32) * 32, 0, x->sa_stream>>>(sa);
      const cudaError_t ce = cudaStreamEndCapture(x->sa_stream, &graph);
      graphed = ge == HEDDLE_OK && ce == cudaSuccess && graph &&
                cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    }
    cudaGetLastError();
    x->launches = l0;
    if (!graphed) {
      if (exec) cudaGraphExecDestroy(exec);
      exec = nullptr;
    }
  }
  for (int it = 0; it < nit; ++it) {
    if (graphed) {
      if (cudaGraphLaunch(exec, s) != cudaSuccess) { e = HEDDLE_E_CUDA; break; }
      x->launches += 3;
    } else {
      k9_perturb<<<(P + 127) / 128, 128, 0, s>>>(sa);
      x->launches++;
      e = evaluate(sa.prop_deg, sa.prop_m, s);
      if (e != HEDDLE_OK) break;
      k9_accept<<<1, ((P + 31) / 32) * 32, 0, s>>>(sa);
      x->launches++;
    }
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  if (e != HEDDLE_OK) return e;
  x->solved = false;   // the workspace holds the last proposals' rows, not a caller's solve
  if (O->iterations) *O->iterations = nit;
  return cudaGetLastError() == cudaSuccess ? HEDDLE_OK : HEDDLE_E_CUDA;
}

}  // extern "C"

#ifdef HEDDLE_UNITY   // debug / bounds-checked build: one translation unit
#include "inst_k2.cu"
#include "inst_k35.cu"
#include "inst_k4.cu"
#include "inst_k8.cu"
#endif
