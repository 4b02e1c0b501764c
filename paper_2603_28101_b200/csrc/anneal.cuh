// K9 -- device-resident sort-initialised simulated annealing (§6.2, Alg. 2).
//
// P independent chains of Alg. 2 walk over sorted MP-degree allocations; every
// iteration is three stream-ordered steps with no host round trip:
//   k9_perturb  one thread per chain: Alg. 2 Perturb -- split / merge / redistribute
//               (R13) -- into the proposal row, the worker count m_b changes (R14);
//   solve       ONE ragged launch over all P proposals (heddle_place_problem.ms): the
//               PresortedDP makespans of line 8;
//   k9_accept   one thread per chain: the Metropolis rule of lines 9-12, the best-so-far
//               of lines 13-14 and the cooling T <- alpha T of line 16, stop at T <= eps.
// The randomness is an input (R16): per chain and iteration the uniforms (kind, first pick,
// second pick, acceptance) are consumed by the fixed protocol of allocator.py / oracle/sa.py:
// the kind order starts at floor(3 u0) and falls through split -> merge -> redistribute when a
// move is inapplicable; candidates are listed in descending degree order and picked by
// floor(u * count).  A chain's state is its count per profile degree, so every move is O(D).
#pragma once
#include <cstdint>

#include "dp_batched.cuh"

namespace hp {

constexpr int kK9MaxD = 16;   // profile degrees handled by the move logic

struct AnnealArgs {
  int P, M, n, D;             // chains, row stride (m_max), trajectories, profile degrees
  int m_min, m_max;
  const int* deg_desc;        // [D] profile degrees, descending
  const double* u;            // [P][iters][4]
  int iters;
  double cooling;
  int* cur_deg;               // [P][M] current sorted degrees
  int* cur_m;                 // [P]
  int* prop_deg;              // [P][M] proposal (solved by the DP)
  int* prop_m;                // [P]
  double* C;                  // [P] current makespan
  double* T;                  // [P] temperature
  double* eps;                // [P] stop threshold eps_frac * T0
  int* live;                  // [P] T > eps
  double* best;               // [P] best makespan
  int* best_deg;              // [P][M]
  int* best_m;                // [P]
  double* trace_c;            // [P][iters + 1] current makespan after each iteration (col 0: start)
  int* accepted;              // [P][iters] 1 if the iteration's proposal was accepted
  int* it;                    // iteration counter (device; advanced by k9_accept)
  const void* obj;            // [P] makespans of the proposals (solve / objective output)
  int obj_kind;               // 0 float, 1 double, 2 uint32, 3 uint64
};

__device__ __forceinline__ double obj_value(const AnnealArgs& s, int c) {
  switch (s.obj_kind) {
    case 0: { const float v = reinterpret_cast<const float*>(s.obj)[c]; return (double)v; }
    case 1: return reinterpret_cast<const double*>(s.obj)[c];
    case 2: { const uint32_t v = reinterpret_cast<const uint32_t*>(s.obj)[c];
              return v == 0xFFFFFFFFu ? __longlong_as_double(0x7ff0000000000000ll) : (double)v; }
    default: { const uint64_t v = reinterpret_cast<const uint64_t*>(s.obj)[c];
               return v == ~0ull ? __longlong_as_double(0x7ff0000000000000ll) : (double)v; }
  }
}

// floor(u * count) clamped to count - 1 (the protocol's pick(seq, u))
__device__ __forceinline__ int pick_index(double u, int count) {
  const int t = (int)(u * (double)count);
  return t < count - 1 ? t : count - 1;
}

// counts per degree index (descending degrees) <- sorted row of m entries; -1 for unknown
__device__ __forceinline__ int degree_index(const AnnealArgs& s, int d) {
  for (int q = 0; q < s.D; ++q)
    if (s.deg_desc[q] == d) return q;
  return -1;
}

// Alg. 2 Perturb under the fixed protocol.  cnt: counts per degree index, m: worker count.
// Returns true if a move applied (cnt / m updated).
__device__ bool perturb_counts(const AnnealArgs& s, int (&cnt)[kK9MaxD], int& m, const double* u4) {
  const int D = s.D;
  const int first = min((int)(u4[0] * 3.0), 2);
  for (int t = 0; t < 3; ++t) {
    const int kind = (first + t) % 3;
    if (kind == 0) {   // split: d -> d/2 + d/2 (d even, d/2 allowed); m + 1 <= m_max
      if (m + 1 > s.m_max) continue;
      int cand[kK9MaxD], nc = 0;
      for (int q = 0; q < D; ++q) {
        const int d = s.deg_desc[q];
        if (cnt[q] > 0 && d % 2 == 0 && degree_index(s, d / 2) >= 0) cand[nc++] = q;
      }
      if (nc == 0) continue;
      const int q = cand[pick_index(u4[1], nc)];
      cnt[q] -= 1;
      cnt[degree_index(s, s.deg_desc[q] / 2)] += 2;
      m += 1;
      return true;
    } else if (kind == 1) {   // merge: d + d -> 2d (2d allowed); m - 1 >= m_min
      if (m - 1 < s.m_min) continue;
      int cand[kK9MaxD], nc = 0;
      for (int q = 0; q < D; ++q) {
        const int d = s.deg_desc[q];
        if (cnt[q] >= 2 && degree_index(s, 2 * d) >= 0) cand[nc++] = q;
      }
      if (nc == 0) continue;
      const int q = cand[pick_index(u4[1], nc)];
      cnt[q] -= 2;
      cnt[degree_index(s, 2 * s.deg_desc[q])] += 1;
      m -= 1;
      return true;
    } else {   // redistribute: (v, w) -> another allowed (x, y), x >= y, x + y = v + w
      // pairs (v, w) over the distinct present values, v >= w, in descending order, that have an
      // alternative; alternatives (x, y) with x over the degrees descending, then y descending
      auto n_alts = [&](int v, int w) {
        int k = 0;
        for (int a = 0; a < D; ++a)
          for (int b = 0; b < D; ++b) {
            const int x = s.deg_desc[a], y = s.deg_desc[b];
            if (x >= y && x + y == v + w && !(x == v && y == w)) ++k;
          }
        return k;
      };
      int npairs = 0;
      for (int a = 0; a < D; ++a)
        for (int b = a; b < D; ++b) {
          if (cnt[a] == 0 || cnt[b] == 0 || (a == b && cnt[a] < 2)) continue;
          if (n_alts(s.deg_desc[a], s.deg_desc[b]) > 0) ++npairs;
        }
      if (npairs == 0) continue;
      const int pk = pick_index(u4[1], npairs);
      int seen = 0;
      for (int a = 0; a < D; ++a)
        for (int b = a; b < D; ++b) {
          if (cnt[a] == 0 || cnt[b] == 0 || (a == b && cnt[a] < 2)) continue;
          const int v = s.deg_desc[a], w = s.deg_desc[b];
          const int na = n_alts(v, w);
          if (na == 0) continue;
          if (seen++ != pk) continue;
          const int ak = pick_index(u4[2], na);
          int k = 0;
          for (int xa = 0; xa < D; ++xa)
            for (int yb = 0; yb < D; ++yb) {
              const int x = s.deg_desc[xa], y = s.deg_desc[yb];
              if (!(x >= y && x + y == v + w && !(x == v && y == w))) continue;
              if (k++ != ak) continue;
              cnt[a] -= 1;
              cnt[b] -= 1;
              cnt[xa] += 1;
              cnt[yb] += 1;
              return true;
            }
        }
      return false;   // unreachable
    }
  }
  return false;
}

__device__ __forceinline__ void counts_of(const AnnealArgs& s, const int* row, int m, int (&cnt)[kK9MaxD]) {
  for (int q = 0; q < kK9MaxD; ++q) cnt[q] = 0;
  for (int j = 0; j < m; ++j) {
    const int q = degree_index(s, row[j]);
    if (q >= 0) cnt[q] += 1;
  }
}

__device__ __forceinline__ void write_row(const AnnealArgs& s, const int (&cnt)[kK9MaxD], int* row) {
  int j = 0;
  for (int q = 0; q < s.D; ++q)
    for (int r = 0; r < cnt[q]; ++r) row[j++] = s.deg_desc[q];   // sorted descending
  for (; j < s.M; ++j) row[j] = s.deg_desc[0];                    // padding (never read: j >= m_b)
}

// Alg. 2 lines 6-7: the proposal of every live chain (others re-submit their current state).
__global__ void k9_perturb(AnnealArgs s) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= s.P) return;
  const int it = *s.it;
  const int* cur = s.cur_deg + (int64_t)c * s.M;
  int* prop = s.prop_deg + (int64_t)c * s.M;
  int m = s.cur_m[c];
  int cnt[kK9MaxD];
  counts_of(s, cur, m, cnt);
  const int m0 = m;
  if (s.live[c] && it < s.iters) {
    perturb_counts(s, cnt, m, s.u + ((int64_t)c * s.iters + it) * 4);
    if (m > s.n) {   // proposals beyond n workers are infeasible: stay (allocator.anneal)
      counts_of(s, cur, m0, cnt);
      m = m0;
    }
  }
  write_row(s, cnt, prop);
  s.prop_m[c] = m;
}

// Alg. 2 lines 8-16 after the ragged solve of the proposals; one block, one thread per chain.
__global__ void k9_accept(AnnealArgs s) {
  const int c = threadIdx.x;
  const int it = *s.it;
  if (c < s.P) {
    int acc = 0;
    if (s.live[c] && it < s.iters) {
      const double Cn = obj_value(s, c);
      const double d = Cn - s.C[c];
      acc = (d < 0.0) || (s.u[((int64_t)c * s.iters + it) * 4 + 3] < exp(-d / s.T[c]));
      if (acc) {
        for (int j = 0; j < s.M; ++j) s.cur_deg[(int64_t)c * s.M + j] = s.prop_deg[(int64_t)c * s.M + j];
        s.cur_m[c] = s.prop_m[c];
        s.C[c] = Cn;
        if (Cn < s.best[c]) {
          s.best[c] = Cn;
          for (int j = 0; j < s.M; ++j) s.best_deg[(int64_t)c * s.M + j] = s.prop_deg[(int64_t)c * s.M + j];
          s.best_m[c] = s.prop_m[c];
        }
      }
      s.T[c] *= s.cooling;
      s.live[c] = s.T[c] > s.eps[c];
    }
    if (it < s.iters) {
      if (s.trace_c) s.trace_c[(int64_t)c * (s.iters + 1) + it + 1] = s.C[c];
      if (s.accepted) s.accepted[(int64_t)c * s.iters + it] = acc;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *s.it = it + 1;
}

// start of the walk (lines 1-4): C = T = the initial makespans, eps = eps_frac * T0, best = start
__global__ void k9_start(AnnealArgs s, double eps_frac) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c == 0) *s.it = 0;
  if (c >= s.P) return;
  const double C0 = obj_value(s, c);
  s.C[c] = C0;
  s.T[c] = C0;
  s.eps[c] = eps_frac * C0;
  s.live[c] = C0 > eps_frac * C0;
  s.best[c] = C0;
  for (int j = 0; j < s.M; ++j) s.best_deg[(int64_t)c * s.M + j] = s.cur_deg[(int64_t)c * s.M + j];
  s.best_m[c] = s.cur_m[c];
  if (s.trace_c) s.trace_c[(int64_t)c * (s.iters + 1)] = C0;
}

}  // namespace hp
